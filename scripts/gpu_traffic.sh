# full-size DRAM traffic of the bench's collide launch (ncu), fp64 and fp32 storage
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for prec in fp64 fp32; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    --clock-control none -k regex:collide -s 3 -c 1 --csv \
    python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu-baseline --precision $prec 2>/dev/null | grep "^\"" \
    > gpurun_out/traffic_$prec.csv
  echo "$prec $?"
done
