# x-pair fp32 kernel (wrap-aware fast path): parity + register-cap sweep, short and sustained
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fastpath.py "tests/test_gpu_parity.py::test_full_fd_fused_kernel_equals_two_pass" -m gpu -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2c_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for v in scalar xp4 xp5 xp6; do
  case $v in scalar) export LBM_XPAIR=0; unset LBM_CUBOID_LIB;; xp4) export LBM_XPAIR=1; unset LBM_CUBOID_LIB;; *) export LBM_XPAIR=1; export LBM_CUBOID_LIB=$PWD/build/variants/lib_$v.so;; esac
  for st in 20 600; do
    timeout 300 python bench.py --steps $st --warmup 5 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/r2c_bench_${v}_s${st}.log 2>&1
    echo "fp32 $v steps=$st: $(summ gpurun_out/r2c_bench_${v}_s${st}.log)"
  done
done
unset LBM_CUBOID_LIB; export LBM_XPAIR=1
cat > /tmp/one.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import paper_2107_14774_b200 as P, synth
w = synth.CONFIGS["weak"].scaled(nx=512, ny=512, nz=64, precision=1)
g = P.Lattice(**w.params(), graphs=1)
rho, u = synth.initial_fields(w)
g.init_fields(rho, u); g.step(3); g.sync(); print("ok")
PY
python /tmp/one.py > gpurun_out/r2c_one.log 2>&1 && \
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio --clock-control none -k regex:collide_stream -s 1 -c 1 --csv python /tmp/one.py > gpurun_out/r2c_ncu_xp.csv 2>&1; echo "ncu $?"
