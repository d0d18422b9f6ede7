# round-2 ncu captures (--set full) of the collide-stream kernels on 512x512x64;
# the reports are summarised to CSV on the box (the .ncu-rep files exceed the copy-back limit)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof_r2
NCU="ncu -f --set full --clock-control none --import-source on -k regex:k_collide_stream -s 1 -c 1"
run() {  # name, env..., args
  n=$1; shift
  env "$@" python scripts/prof_one.py $ARGS > gpurun_out/prof_r2/$n.plain.log 2>&1 && \
  env "$@" $NCU -o /tmp/$n python scripts/prof_one.py $ARGS > gpurun_out/prof_r2/$n.ncu.log 2>&1
  echo "$n $?"
  ncu -i /tmp/$n.ncu-rep --page details --csv > gpurun_out/prof_r2/${n}_details.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page raw --csv > /tmp/${n}_raw.csv 2>/dev/null
  python - "$n" <<'PY'
import csv, sys, io
n = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/{n}_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "l1tex__t_bytes_pipe_lsu_mem_local",
        "smsp__average_warp_latency_issue_stalled", "sm__pipe_fp64_cycles_active")
with open(f"gpurun_out/prof_r2/{n}_raw_selected.csv", "w") as fh:
    for h, u, v in zip(hdr, units, vals):
        if any(h.startswith(w) for w in want):
            fh.write(f"{h},{u},{v}\n")
PY
}
ARGS="fp64" run paper_fp64
ARGS="fp32" run paper_fp32
ARGS="fp64 full_fd_lag" run fd_lag_fp64
ARGS="fp64" run tma_fp64 LBM_TMA=1
ARGS="fp32" run tma_fp32 LBM_TMA=1
ls -la gpurun_out/prof_r2; du -sh gpurun_out
