cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,power.draw.instant,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 50 > gpurun_out/fp64_clocks.csv &
SMI=$!
./build/fp64_peak > gpurun_out/fp64_peak.log 2>&1; echo "peak exit $?"
kill $SMI
cat gpurun_out/fp64_peak.log
awk -F, '$2+0>300 {print $1}' gpurun_out/fp64_clocks.csv | sort | uniq -c | sort -rn | head -5
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_conversion_pred_on.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for p in fp64 fp32; do
  B="python bench.py --precision $p --steps 3 --warmup 2 --nz-per-gpu 64 --no-e2e --no-cpu-baseline"
  timeout 300 $B > gpurun_out/plain_$p.log 2>&1 && timeout 900 ncu --metrics $M --clock-control none -k regex:collide -s 2 -c 1 --csv --log-file gpurun_out/ncu_dp_$p.csv $B > gpurun_out/ncu_dp_$p.log 2>&1
  echo "ncu $p exit $?"
done
