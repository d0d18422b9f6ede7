# the GPU suite and smoke on the final commit of round 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3i
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3i/gpu_tests.log 2>&1; echo "gpu tests $?"; tail -2 gpurun_out/r3i/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
