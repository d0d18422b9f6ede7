cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/w_smoke.log 2>&1; echo "smoke $?"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/w_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/w_tests.log
timeout 600 python scripts/wall_cost.py > gpurun_out/wall_cost2.log 2>&1; timeout 600 python scripts/wall_cost.py --precision fp32 >> gpurun_out/wall_cost2.log 2>&1; cat gpurun_out/wall_cost2.log
for args in "" "--precision fp32" "--workload cavity100" "--workload shear"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $args > gpurun_out/w_bench.log 2>&1
  tail -1 gpurun_out/w_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', '$args', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
