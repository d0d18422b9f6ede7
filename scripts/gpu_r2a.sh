# round-2 regression: new tests first, then the whole GPU suite, then quick benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke $?"
timeout 900 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_singular_aa_lid.py tests/test_gpu_p2p.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_new_tests.log 2>&1; echo "new tests $?"; tail -3 gpurun_out/r2_new_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2_tests.log
for args in "" "--corrections full_fd" "--precision fp32"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $args > gpurun_out/r2_bench.log 2>&1
  tail -1 gpurun_out/r2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', '$args', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
