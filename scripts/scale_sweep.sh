# Weak and strong scaling on the GPUs of one box, both halo modes (run when more
# than one GPU is available):  bash scripts/scale_sweep.sh [max_gpus] > scale.jsonl
# DRY_RUN=1: no GPU -- every bench.py call gets --dry-run (plan + gloo aggregation
# check), so the launch logic of the sweep runs on a CPU (tests/test_bench_dryrun.py).
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
MAX=${1:-$(nvidia-smi -L | wc -l)}
PORT=${PORT:-29600}
DRY=""
[ -n "$DRY_RUN" ] && DRY="--dry-run"
run() {  # n, extra bench args...
  local n=$1; shift
  PORT=$((PORT + 1))
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $DRY "$@" | tail -1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
      --master-port $PORT bench.py --gpus "$n" --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $DRY "$@" 2>/dev/null | tail -1
  fi
}
for n in 1 2 4 8; do
  [ "$n" -gt "$MAX" ] && break
  run $n --halo auto                          # weak, 512^3 per GPU, NCCL halo (in-kernel wrap at n = 1)
  run $n --halo p2p                           # weak, fused peer-memory halo
  if [ "$n" = 1 ]; then
    run 1 --workload strong --streaming aa    # strong 1024x1024x512 fits one GPU only in place (116 GB)
  else
    run $n --workload strong --halo auto
    run $n --workload strong --halo p2p
  fi
done
