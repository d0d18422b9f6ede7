# experiment: FULL_FD TMA ring densities as three partial sums (speed only; not bitwise with the other paths)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3g
python scripts/fd_tma_variants.py run base ring3 base ring3 > gpurun_out/r3g/variants.jsonl 2>&1
cut -c1-110 gpurun_out/r3g/variants.jsonl
