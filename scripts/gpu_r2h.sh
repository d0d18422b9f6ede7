cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fd_lag.py tests/test_gpu_parity.py -k "fd or lag or FD" -m gpu -q -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2h_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
for c in full_fd_lag; do for p in fp64 fp32; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --corrections $c --precision $p > gpurun_out/r2h_bench_${c}_${p}.log 2>&1
  echo "$c $p: $(summ gpurun_out/r2h_bench_${c}_${p}.log)"
done; done
timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --corrections full_fd_lag > gpurun_out/r2h_bench_lag_200.log 2>&1; echo "lag fp64 200 steps: $(summ gpurun_out/r2h_bench_lag_200.log)"
