# final check of bench.py (default line and the reference arm) after the late bench.py changes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3f
python bench.py > gpurun_out/r3f/bench_default.jsonl 2> gpurun_out/r3f/bench_default.err; echo "bench $?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3f/bench_reference.jsonl 2> gpurun_out/r3f/bench_reference.err; echo "reference $?"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
