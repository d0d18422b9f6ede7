# randomised parity stress on fresh draws (seed offset 2) against the final build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3c
LBM_FUZZ_SEED_OFFSET=2 LBM_FUZZ_CASES=600 LBM_FUZZ_SLAB_CASES=40 LBM_FUZZ_FDTMA_CASES=100 LBM_FUZZ_SHAPE_CASES=60 \
  timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -rs > gpurun_out/r3c/fuzz_stress_seed2.log 2>&1
echo "fuzz $?"; tail -3 gpurun_out/r3c/fuzz_stress_seed2.log
