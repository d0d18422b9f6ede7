# full GPU suite after the FULL_FD TMA kernel became the default where it applies; FD benches
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2x_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2x_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2x_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2x_$n.log)"; }
run fd64 --steps 50 --corrections full_fd
run fd32 --steps 50 --corrections full_fd --precision fp32
run fd64_200 --steps 200 --corrections full_fd
