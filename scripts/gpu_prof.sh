# GPU round-trip: parity tests, bench, ncu launch list + one full capture of the collide kernel
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"
tail -3 gpurun_out/gpu_tests.log
BENCH="python bench.py --steps 20 --warmup 5"
timeout 600 $BENCH > gpurun_out/bench_$TAG.log 2>&1 && echo "bench ok" && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $BENCH > gpurun_out/ncu_launches.log 2>&1
echo "launch list exit $?"
tail -1 gpurun_out/bench_$TAG.log
PROF="python bench.py --steps 3 --warmup 2 --nz-per-gpu 64 --no-e2e --no-cpu-baseline"
timeout 300 $PROF > gpurun_out/prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:collide -s 2 -c 1 -o gpurun_out/prof_cs_$TAG $PROF > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
tail -2 gpurun_out/ncu_full.log
