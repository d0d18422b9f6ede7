set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fd_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_fd" > gpurun_out/fd_tests.log 2>&1
echo "fd tests exit $?"
tail -5 gpurun_out/fd_tests.log
for fused in 1 0; do
  LBM_FD_FUSED=$fused timeout 300 python bench.py --steps 10 --warmup 3 --corrections full_fd --no-e2e --no-cpu-baseline > gpurun_out/bench_fd_fused$fused.log 2>&1
  echo "bench fd fused=$fused exit $?"
  tail -1 gpurun_out/bench_fd_fused$fused.log | cut -c1-300
done
