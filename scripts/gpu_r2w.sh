# FULL_FD TMA kernel: persistent vs one CTA per tile (+ the kernel's GPU tests)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fd_tma.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2w_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2w_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2w_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2w_$n.log)"; }
for prec in fp64 fp32; do
  LBM_FD_TMA=1 LBM_FD_TMA_PERSIST=1 run pers_$prec --steps 20 --corrections full_fd --precision $prec
  LBM_FD_TMA=1 LBM_FD_TMA_PERSIST=0 run tile_$prec --steps 20 --corrections full_fd --precision $prec
done
