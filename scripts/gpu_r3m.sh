# final evidence of the last build: GPU suite, smoke, bench-launch traffic (recorded on the box so the
# bench line that follows resolves roofline.traffic), default bench + reference arm, launch list, ncu full
cd $GRAFT_REPO_ROOT
O=gpurun_out/final3; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "gpu tests $?"; tail -1 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for p in fp64:double fp32:float; do pr=${p%%:*}; t=${p##*:}
  python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision $pr > $O/plain_$pr.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --precision $pr > $O/ncu_traffic_$pr.csv 2>&1; echo "ncu $pr $?"
  python scripts/ncu_traffic_update.py $O/ncu_traffic_$pr.csv --workload 'config5-weak-tgv-512^3-per-gpu' --precision $pr --kernel "k_collide_stream_paper_shape<$t,512,512>" --nodes 134217728 | cut -c1-200
done
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python bench.py > $O/bench_default.jsonl 2> $O/bench_default.err; echo "bench $?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.jsonl 2> $O/bench_reference.err; echo "reference $?"
python bench.py --steps 50 --precision fp32 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > $O/bench_fp32.jsonl
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launches $?"
for prec in fp64 fp32; do
  python scripts/prof_one.py $prec > /dev/null 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:k_collide_stream -s 1 -c 1 -o /tmp/shape_$prec python scripts/prof_one.py $prec > $O/ncu_full_$prec.log 2>&1
  echo "ncu full $prec $?"
  ncu -i /tmp/shape_$prec.ncu-rep --page details --csv > $O/shape_${prec}_details.csv 2>/dev/null
  ncu -i /tmp/shape_$prec.ncu-rep --page raw --csv > $O/shape_${prec}_raw.csv 2>/dev/null
done
