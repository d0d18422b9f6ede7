# final round-2 evidence for this build (after the fp32 AA launch bound): GPU suite, smoke, bench line, launch list of the
# bench command, DRAM traffic of the bench launch (fp64, fp32), ncu full of the shape kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/gpu_tests.log 2>&1; echo "gpu tests $?"; tail -2 gpurun_out/final2/gpu_tests.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final2/bench_default.jsonl 2> gpurun_out/final2/bench_default.err; echo "bench $?"
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final2/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final2/ncu_launches.log 2>&1; echo "launches $?"
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/final2/plain64.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/final2/ncu_traffic_fp64.csv 2>&1; echo "ncu64 $?"
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/final2/plain32.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/final2/ncu_traffic_fp32.csv 2>&1; echo "ncu32 $?"
for prec in fp64 fp32; do
  python scripts/prof_one.py $prec > /dev/null 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:k_collide_stream -s 1 -c 1 -o /tmp/shape_$prec python scripts/prof_one.py $prec > gpurun_out/final2/ncu_full_$prec.log 2>&1
  echo "ncu full $prec $?"
  ncu -i /tmp/shape_$prec.ncu-rep --page details --csv > gpurun_out/final2/shape_${prec}_details.csv 2>/dev/null
  ncu -i /tmp/shape_$prec.ncu-rep --page raw --csv > gpurun_out/final2/shape_${prec}_raw.csv 2>/dev/null
done
du -sh gpurun_out
for a in "--precision fp32" "--workload cavity100 --precision fp32" "" "--workload cavity100"; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --streaming aa $a 2>/dev/null | tail -1 >> gpurun_out/final2/aa_lines.jsonl
done
cut -c1-200 gpurun_out/final2/aa_lines.jsonl
