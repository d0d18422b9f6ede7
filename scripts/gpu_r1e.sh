cd $GRAFT_REPO_ROOT
for wl in cavity100 cavity1000 shear tgv; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.log 2>&1; echo "$wl exit $?"
  tail -1 gpurun_out/bench_$wl.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],round(d['value']),d['ms_per_step'],round(d['roofline']['frac'],3),d['e2e']['value'] if d['e2e'] else None)"
done
B="python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/b_full.log 2>&1 && \
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:collide -s 4 -c 2 --csv --log-file gpurun_out/ncu_full_traffic.csv $B > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
tail -8 gpurun_out/ncu_full_traffic.csv
