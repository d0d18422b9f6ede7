# tracing + overlap timeline, full GPU suite, default bench, ncu traffic capture of the bench launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_trace.py -m gpu -q -p no:cacheprovider > gpurun_out/r2f_trace_tests.log 2>&1; echo "trace tests $?"; tail -2 gpurun_out/r2f_trace_tests.log
timeout 300 python scripts/overlap_trace.py 6 > gpurun_out/overlap_trace.json 2> gpurun_out/overlap_trace.err; echo "overlap $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/overlap_trace.json"))
for r in d["runs"]:
    for s in r["steps"]:
        print(r["halo"], {k: (round(v, 3) if isinstance(v, float) else [round(x, 3) for x in v] if isinstance(v, list) else v) for k, v in s.items()})
PY
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "gpu tests $?"; tail -3 gpurun_out/r2f_tests.log
timeout 600 python bench.py > gpurun_out/r2f_bench_default.log 2>&1; echo "bench $?"; tail -1 gpurun_out/r2f_bench_default.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r2f_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_traffic_fp64.csv 2>&1; echo "ncu64 $?"
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/r2f_plain32.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/ncu_traffic_fp32.csv 2>&1; echo "ncu32 $?"
