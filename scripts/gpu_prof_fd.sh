# ncu --set full of the FULL_FD collide kernels (fused and two-pass) on 512x512x64
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PROF="python bench.py --steps 3 --warmup 2 --nz-per-gpu 64 --no-e2e --no-cpu-baseline --corrections full_fd"
LBM_FD_FUSED=1 timeout 300 $PROF > gpurun_out/prof_fd_plain.log 2>&1 && \
  LBM_FD_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide_stream_fd -s 2 -c 1 -o gpurun_out/prof_fd_fused $PROF > gpurun_out/ncu_fd_fused.log 2>&1
echo "ncu fused exit $?"
LBM_FD_FUSED=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collide_stream_paper|k_density" -s 4 -c 2 -o gpurun_out/prof_fd_twopass $PROF > gpurun_out/ncu_fd_twopass.log 2>&1
echo "ncu twopass exit $?"
