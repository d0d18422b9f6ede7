# x-pair fp32 kernel: parity, A/B bench (short + sustained), ncu instruction counts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_singular_aa_lid.py "tests/test_gpu_parity.py::test_full_fd_fused_kernel_bitwise_equal_two_pass" "tests/test_gpu_parity.py::test_checkpoint_resume_is_exact" -m gpu -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2b_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for xp in 0 1; do
  for st in 20 1000; do
    LBM_XPAIR=$xp timeout 300 python bench.py --steps $st --warmup 5 --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/r2b_bench_xp${xp}_s${st}.log 2>&1
    echo "fp32 xpair=$xp steps=$st: $(summ gpurun_out/r2b_bench_xp${xp}_s${st}.log)"
  done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_fp64.log 2>&1; echo "fp64: $(summ gpurun_out/r2b_bench_fp64.log)"
# instruction counts of both fp32 kernels on 512x512x64 (one launch each)
cat > /tmp/one.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import paper_2107_14774_b200 as P, synth
w = synth.CONFIGS["weak"].scaled(nx=512, ny=512, nz=64, precision=1)
g = P.Lattice(**w.params(), graphs=1)
rho, u = synth.initial_fields(w)
g.init_fields(rho, u); g.step(3); g.sync(); print("ok")
PY
for xp in 0 1; do
  LBM_XPAIR=$xp python /tmp/one.py > gpurun_out/r2b_one_$xp.log 2>&1 && \
  LBM_XPAIR=$xp ncu --metrics smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:collide_stream -s 1 -c 1 --csv python /tmp/one.py > gpurun_out/r2b_ncu_xp$xp.csv 2>&1
  echo "ncu $xp rc=$?"
done
