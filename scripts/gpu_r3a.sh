# FULL_FD TMA kernel: early stage release (LBM_FD_TMA_EARLY) A/B, parity of the variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3a
for v in early_r200 early; do
  LBM_CUBOID_LIB=$PWD/varbuild/lib_fdtma_$v.so timeout 900 python -m pytest tests/test_gpu_fd_tma.py -q -x -p no:cacheprovider > gpurun_out/r3a/test_$v.log 2>&1; echo "tests $v $?"; tail -1 gpurun_out/r3a/test_$v.log
done
python scripts/fd_tma_variants.py run base early early_m32_2 early_r200 base_r200 > gpurun_out/r3a/variants.jsonl 2>&1
python scripts/fd_tma_variants.py run base early_r200 early early_m32_2 >> gpurun_out/r3a/variants.jsonl 2>&1
cat gpurun_out/r3a/variants.jsonl | cut -c1-120
