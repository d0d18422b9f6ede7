# ncu --set full with SASS source of the FULL_FD TMA kernel (fp64, fp32) on 512x512x64: per-instruction stall attribution
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof_r3
NCU="ncu -f --set full --clock-control none --import-source on -k regex:k_collide_stream_fd -s 1 -c 1"
run() {  # name, env...
  n=$1; shift
  env "$@" python scripts/prof_one.py $ARGS > gpurun_out/prof_r3/$n.plain.log 2>&1 && \
  env "$@" $NCU -o /tmp/$n python scripts/prof_one.py $ARGS > gpurun_out/prof_r3/$n.ncu.log 2>&1
  echo "$n $?"
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/prof_r3/${n}_raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source sass > /tmp/${n}_sass.csv 2>/dev/null
  gzip -c /tmp/${n}_sass.csv > gpurun_out/prof_r3/${n}_sass.csv.gz
}
ARGS="fp64 full_fd" run fdtma_fp64 LBM_FD_TMA=1
ARGS="fp32 full_fd" run fdtma_fp32 LBM_FD_TMA=1
