# TMA kernel: probe (subprocesses), tests, bench A/B over variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/tma_probe.py > gpurun_out/r2e_probe.log 2>&1; cat gpurun_out/r2e_probe.log
if grep -q "rc=1\|TIMEOUT" gpurun_out/r2e_probe.log; then echo "probe failed"; exit 0; fi
timeout 600 python -m pytest tests/test_gpu_tma.py tests/test_gpu_fastpath.py -m gpu -q -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2e_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -2 $1; }
run() { # name prec env...
  n=$1; p=$2; shift 2
  for st in 20 600; do
    env "$@" timeout 300 python bench.py --steps $st --warmup 5 --no-e2e --no-cpu-baseline --precision $p > gpurun_out/r2e_${n}_${p}_s${st}.log 2>&1
    echo "$n $p steps=$st: $(summ gpurun_out/r2e_${n}_${p}_s${st}.log)"
  done
}
for p in fp64 fp32; do
  run notma $p LBM_TMA=0
  run tma $p LBM_TMA=1
  run tma_m3 $p LBM_CUBOID_LIB=$PWD/build/variants/lib_tma_m3.so
done
run tma_wb1 fp64 LBM_CUBOID_LIB=$PWD/build/variants/lib_tma_wb1.so
run tma_s2 fp32 LBM_CUBOID_LIB=$PWD/build/variants/lib_tma_s2.so
