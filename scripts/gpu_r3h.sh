# experiment: L2 prefetch (cp.async.bulk.prefetch.tensor) of the FULL_FD TMA kernel's boxes PF planes ahead
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3h
python scripts/fd_tma_variants.py run base pf1 pf2 pf4 base pf2 pf4 pf1 > gpurun_out/r3h/variants.jsonl 2>&1
cut -c1-110 gpurun_out/r3h/variants.jsonl
