cd $GRAFT_REPO_ROOT
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
for args in "" "--precision fp32" "--corrections full_fd_lag" "--corrections full_fd_lag --precision fp32" "--corrections full_fd"; do
  n=$(echo "$args" | tr ' -' '__')
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $args > gpurun_out/r2j_$n.log 2>&1
  echo "[$args]: $(summ gpurun_out/r2j_$n.log)"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2j_again.log 2>&1; echo "[default again]: $(summ gpurun_out/r2j_again.log)"
timeout 900 python -m pytest tests/test_gpu_fd_lag.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2j_tests.log
