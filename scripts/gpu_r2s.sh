# plane-shape specialised kernels: bitwise tests, A/B benches (short and sustained), instruction counts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shape.py tests/test_gpu_fastpath.py -m gpu -q -p no:cacheprovider > gpurun_out/r2s_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2s_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2s_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2s_$n.log)"; }
for spec in 1; do
  export LBM_SHAPE_SPEC=$spec
  run fp32_s20_spec$spec --steps 20 --precision fp32
  run fp32_s600_spec$spec --steps 600 --precision fp32
  run fp64_s20_spec$spec --steps 20
  run lag_s50_spec$spec --steps 50 --corrections full_fd_lag
  run lag32_s50_spec$spec --steps 50 --corrections full_fd_lag --precision fp32
  run cav32_spec$spec --workload cavity100 --steps 50 --precision fp32
done
unset LBM_SHAPE_SPEC
run fp64_s1000 --steps 1000
run fp32_s1000 --steps 1000 --precision fp32
python scripts/prof_one.py fp32 > /dev/null 2>&1 && ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,launch__registers_per_thread --clock-control none -k regex:k_collide_stream -s 1 -c 1 --csv python scripts/prof_one.py fp32 2>&1 | grep -E "inst_executed|time_duration|registers" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
