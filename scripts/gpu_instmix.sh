# executed-instruction mix per node of the collide kernel (ncu), 512x512x64, for bench args "$@"
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
M=smsp__sass_thread_inst_executed.sum
for op in dfma dadd dmul integer conversion memory control uniform; do M=$M,smsp__sass_thread_inst_executed_op_${op}_pred_on.sum; done
timeout 600 ncu --metrics $M,gpu__time_duration.sum --clock-control none -k regex:collide -s 2 -c 1 --csv python bench.py --steps 3 --warmup 2 --nz-per-gpu 64 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | grep "^\"" | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
iv=h.index('Metric Value'); im=h.index('Metric Name')
for row in r[1:]:
    v=float(row[iv].replace(',',''))
    n=row[im].replace('smsp__sass_thread_inst_executed','inst').replace('_pred_on.sum','')
    print(n, round(v/16777216,1) if 'inst' in n else v)
"
