cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LBM_FUZZ_CASES=2000 LBM_FUZZ_SLAB_CASES=400 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/r2m_fuzz_stress.log 2>&1; echo "fuzz stress $?"; tail -5 gpurun_out/r2m_fuzz_stress.log
