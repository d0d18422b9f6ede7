# experiment: minimum resident CTAs of the AA plane-shape kernels (odd kernel 96 -> 80 / 72 registers)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3j
one() {  # name lib args...
  n=$1; lib=$2; shift 2
  LBM_CUBOID_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --streaming aa "$@" > gpurun_out/r3j/$n.log 2>&1
  tail -1 gpurun_out/r3j/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'variant': '$n', 'args': '$*', 'mlups': round(d['value']), 'frac': round(d['roofline']['frac'],3), 'kernel': d['roofline']['kernel'], 'clocks': d['clocks']}))" >> gpurun_out/r3j/lines.jsonl 2>/dev/null || echo "$n failed" >> gpurun_out/r3j/lines.jsonl
}
for rep in 1 2; do
  for v in base m6 m7; do
    lib=$PWD/varbuild/lib_aa_$v.so; [ $v = base ] && lib=$PWD/paper_2107_14774_b200/liblbm_cuboid.so
    one ${v}_fp32 $lib --precision fp32
    one ${v}_fp64 $lib
  done
done
cut -c1-160 gpurun_out/r3j/lines.jsonl
