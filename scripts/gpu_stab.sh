cd $GRAFT_REPO_ROOT
for f in fig8 fig9 fig10; do
  timeout 1500 python -m studies.stability --study $f --steps 100000 --iters 7 --out gpurun_out/stability_$f.json > gpurun_out/stab_$f.log 2>&1; echo "$f exit $?"
  grep seconds gpurun_out/stability_$f.json
done
