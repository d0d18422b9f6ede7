# experiment: resident CTAs of the fp32 plane-shape collide-stream kernel (78 -> 72 / 64 registers)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3l
one() {  # name lib args...
  n=$1; lib=$2; shift 2
  LBM_CUBOID_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --precision fp32 "$@" > gpurun_out/r3l/$n.log 2>&1
  tail -1 gpurun_out/r3l/$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'variant': '$n', 'args': '$*', 'mlups': round(d['value']), 'frac': round(d['roofline']['frac'],3), 'kernel': d['roofline']['kernel'], 'clocks': d['clocks']}))" >> gpurun_out/r3l/lines.jsonl 2>/dev/null || echo "$n failed" >> gpurun_out/r3l/lines.jsonl
}
for rep in 1 2; do
  for v in base m7 m8; do
    lib=$PWD/varbuild/lib_shape_$v.so; [ $v = base ] && lib=$PWD/paper_2107_14774_b200/liblbm_cuboid.so
    one ${v}_weak $lib --steps 50
    one ${v}_cavity $lib --steps 50 --workload cavity100
  done
done
for v in base m7; do
  lib=$PWD/varbuild/lib_shape_$v.so; [ $v = base ] && lib=$PWD/paper_2107_14774_b200/liblbm_cuboid.so
  one ${v}_soak $lib --steps 600
done
cut -c1-160 gpurun_out/r3l/lines.jsonl
