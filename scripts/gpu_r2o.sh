# A/B: round-1 build (build/r1pkg) vs the current build, same harness
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for prec in fp32 fp64; do
  python scripts/ab_time.py build/r1pkg $prec 30
  python scripts/ab_time.py . $prec 30
done
done
python scripts/ab_time.py build/r1pkg fp32 600
python scripts/ab_time.py . fp32 600
(cd build/r1pkg && python prof_r1.py fp32 && ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_collide_stream -s 1 -c 1 --csv python prof_r1.py fp32 2>&1 | grep -E "inst_executed|time_duration" | cut -c1-300)
python scripts/prof_one.py fp32 && ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_collide_stream -s 1 -c 1 --csv python scripts/prof_one.py fp32 2>&1 | grep -E "inst_executed|time_duration" | cut -c1-300
