# TMA kernel: correctness first (short timeout), then bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tma.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2d_tma_tests.log 2>&1; echo "tma tests $?"; tail -5 gpurun_out/r2d_tma_tests.log
timeout 600 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "parity tests $?"; tail -3 gpurun_out/r2d_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for prec in fp64 fp32; do
for tma in 0 1; do
  for st in 20 600; do
    LBM_TMA=$tma timeout 300 python bench.py --steps $st --warmup 5 --no-e2e --no-cpu-baseline --precision $prec > gpurun_out/r2d_bench_${prec}_tma${tma}_s${st}.log 2>&1
    echo "$prec tma=$tma steps=$st: $(summ gpurun_out/r2d_bench_${prec}_tma${tma}_s${st}.log)"
  done
done
done
