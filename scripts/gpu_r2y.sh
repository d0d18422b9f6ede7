# FULL_FD TMA kernel with wall support: its tests + randomised FD-TMA parity, then benches
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fd_tma.py -m gpu -q -p no:cacheprovider > gpurun_out/r2y_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2y_tests.log
LBM_FUZZ_FDTMA_CASES=200 timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k fd_problem_tma > gpurun_out/r2y_fuzz.log 2>&1; echo "fuzz $?"; tail -3 gpurun_out/r2y_fuzz.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2y_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2y_$n.log)"; }
run fd64 --steps 30 --corrections full_fd
run fd32 --steps 30 --corrections full_fd --precision fp32
run cav_fd64 --workload cavity100 --steps 50 --corrections full_fd
LBM_FD_TMA=0 run cav_fd64_2pass --workload cavity100 --steps 50 --corrections full_fd
run cav_fd32 --workload cavity100 --steps 50 --corrections full_fd --precision fp32
LBM_FD_TMA=0 run cav_fd32_2pass --workload cavity100 --steps 50 --corrections full_fd --precision fp32
