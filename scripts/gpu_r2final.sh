# final round-2 evidence for this build: bench line, launch list of the bench command,
# DRAM traffic of the bench launch (fp64, fp32), SASS excerpt of the TMA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_default.jsonl 2> gpurun_out/final/bench_default.err; echo "bench $?"; tail -1 gpurun_out/final/bench_default.jsonl | cut -c1-200
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launches.log 2>&1; echo "launches $?"
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/final/plain64.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_traffic_fp64.csv 2>&1; echo "ncu64 $?"
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/final/plain32.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/final/ncu_traffic_fp32.csv 2>&1; echo "ncu32 $?"
