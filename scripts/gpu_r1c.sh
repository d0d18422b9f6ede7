cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"
tail -4 gpurun_out/gpu_tests.log
mkdir -p results
timeout 900 python -m studies.stability --study fig8 --steps 20000 --iters 5 --out gpurun_out/stab_fig8_quick.json > gpurun_out/stab.log 2>&1; echo "stab exit $?"
tail -5 gpurun_out/stab.log
