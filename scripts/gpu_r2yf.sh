# FULL_FD TMA: tile order x-fastest vs y-fastest (bench twice each, DRAM bytes per launch with ncu)
cd $GRAFT_REPO_ROOT
python scripts/fd_tma_variants.py run > gpurun_out/yf_a.jsonl 2>&1
python scripts/fd_tma_variants.py run > gpurun_out/yf_b.jsonl 2>&1
cat gpurun_out/yf_a.jsonl gpurun_out/yf_b.jsonl | cut -c1-100
for v in xfast yfast; do
  LBM_CUBOID_LIB=varbuild/lib_fdtma_$v.so LBM_FD_TMA=1 ncu -f --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_collide_stream_fd -s 1 -c 1 python scripts/prof_one.py fp64 full_fd 2>&1 | grep -E 'dram__bytes|gpu__time' | sed "s/^/$v /"
done
