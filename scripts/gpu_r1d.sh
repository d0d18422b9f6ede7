cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"
tail -3 gpurun_out/gpu_tests.log
timeout 1200 python -m studies.womersley --out gpurun_out/womersley.json > gpurun_out/wom.log 2>&1; echo "womersley exit $?"
timeout 1800 python -m studies.shallow_cavity --out gpurun_out/shallow_cavity.json > gpurun_out/shallow.log 2>&1; echo "shallow exit $?"
tail -30 gpurun_out/shallow.log
timeout 600 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1; echo "bench32 exit $?"
tail -1 gpurun_out/bench_fp32.log
PROF="python bench.py --precision fp32 --steps 3 --warmup 2 --nz-per-gpu 64 --no-e2e --no-cpu-baseline"
timeout 300 $PROF > gpurun_out/prof32_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:collide -s 2 -c 1 -o gpurun_out/prof_cs32 $PROF > gpurun_out/ncu32.log 2>&1
echo "ncu32 exit $?"
