set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p2p_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_p2p.py -q -x -p no:cacheprovider > gpurun_out/p2p_tests.log 2>&1
echo "p2p tests exit $?"
tail -5 gpurun_out/p2p_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --halo p2p --no-e2e --no-cpu-baseline > gpurun_out/bench_p2p.log 2>&1
echo "bench p2p exit $?"
timeout 300 python bench.py --steps 20 --warmup 5 --halo nccl --no-e2e --no-cpu-baseline > gpurun_out/bench_nccl.log 2>&1
echo "bench nccl exit $?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_auto.log 2>&1
echo "bench auto exit $?"
tail -1 gpurun_out/bench_p2p.log | cut -c1-400
tail -1 gpurun_out/bench_nccl.log | cut -c1-400
tail -1 gpurun_out/bench_auto.log | cut -c1-400
