# FULL_FD TMA kernel with walls (producer-warp fix-ups): tests, randomised parity, benches (periodic + cavity)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fd_tma.py -m gpu -q -p no:cacheprovider > gpurun_out/r2w2_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2w2_tests.log
LBM_FUZZ_FDTMA_CASES=200 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k fd_problem_tma > gpurun_out/r2w2_fuzz.log 2>&1; echo "fuzz $?"; tail -3 gpurun_out/r2w2_fuzz.log
python scripts/fd_tma_variants.py run > gpurun_out/r2w2_var_periodic.jsonl 2>&1; cut -c1-100 gpurun_out/r2w2_var_periodic.jsonl
FD_VARIANT_ARGS="--workload cavity100 --steps 50" python scripts/fd_tma_variants.py run > gpurun_out/r2w2_var_cavity.jsonl 2>&1; cut -c1-100 gpurun_out/r2w2_var_cavity.jsonl
