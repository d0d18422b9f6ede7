cd $GRAFT_REPO_ROOT
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
for v in base minb5 minb6; do
  if [ $v = base ]; then unset LBM_CUBOID_LIB; else export LBM_CUBOID_LIB=$PWD/build/variants/lib_$v.so; fi
  for p in fp64 fp32; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --corrections full_fd_lag --precision $p > gpurun_out/r2i_${v}_${p}.log 2>&1
    echo "$v lag $p: $(summ gpurun_out/r2i_${v}_${p}.log)"
  done
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/r2i_${v}_plain32.log 2>&1
  echo "$v plain fp32: $(summ gpurun_out/r2i_${v}_plain32.log)"
done
