cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shape.py -m gpu -q -p no:cacheprovider > gpurun_out/r2t_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2t_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2t_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2t_$n.log)"; }
for spec in 1 0; do
  export LBM_SHAPE_SPEC=$spec
  run aa_weak64_$spec --steps 50 --streaming aa
  run aa_weak32_$spec --steps 50 --streaming aa --precision fp32
  run aa_cav64_$spec --workload cavity100 --steps 50 --streaming aa
  run aa_cav32_$spec --workload cavity100 --steps 50 --streaming aa --precision fp32
done
