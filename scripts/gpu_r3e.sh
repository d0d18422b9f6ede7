# FULL_FD TMA kernel with the 512x512 plane compiled in (LBM_FD_TMA_SHAPE) A/B + parity; strong config on one GPU (AA fallback)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3e
LBM_CUBOID_LIB=$PWD/varbuild/lib_fdtma_shape.so timeout 900 python -m pytest tests/test_gpu_fd_tma.py -q -x -p no:cacheprovider > gpurun_out/r3e/test_shape.log 2>&1; echo "tests shape $?"; tail -1 gpurun_out/r3e/test_shape.log
python scripts/fd_tma_variants.py run base shape > gpurun_out/r3e/variants.jsonl 2>&1
python scripts/fd_tma_variants.py run shape base >> gpurun_out/r3e/variants.jsonl 2>&1
cut -c1-150 gpurun_out/r3e/variants.jsonl
timeout 900 python bench.py --workload strong --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r3e/strong.log 2>&1; echo "strong $?"; tail -1 gpurun_out/r3e/strong.log | cut -c1-400
