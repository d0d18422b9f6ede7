cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2p_tests.log 2>&1; echo "gpu tests $?"; tail -3 gpurun_out/r2p_tests.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
