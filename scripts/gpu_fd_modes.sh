cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_fd" > gpurun_out/fd_modes_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/fd_modes_tests.log
for prec in fp64 fp32; do for m in 0 1; do
  LBM_FD_FUSED=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --corrections full_fd --precision $prec > gpurun_out/fd_modes_bench.log 2>&1
  tail -1 gpurun_out/fd_modes_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fd', '$prec', 'mode', $m, round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
