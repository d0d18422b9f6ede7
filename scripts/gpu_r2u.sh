# FULL_FD TMA-staged fused kernel: tests, then A/B against the LDG fused kernel and the two-pass path
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fd_tma.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2u_tests.log 2>&1; echo "tests $?"; tail -15 gpurun_out/r2u_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2u_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2u_$n.log)"; }
for prec in fp64 fp32; do
  LBM_FD_TMA=1 run tma_$prec --steps 30 --corrections full_fd --precision $prec
  LBM_FD_FUSED=1 run ldg_$prec --steps 30 --corrections full_fd --precision $prec
  run twopass_$prec --steps 30 --corrections full_fd --precision $prec
done
