# final round-2 build (kernel sources 2a7f5e4edd9cf14c): bench lines of every workload and mode: every workload and mode (profiles/r2/bench_r3d_workloads.jsonl)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 900 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r3d_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r3d_$n.log)"; tail -1 gpurun_out/r3d_$n.log >> gpurun_out/r3d_lines.jsonl; }
rm -f gpurun_out/r3d_lines.jsonl
run weak_fp64 --steps 50
run weak_fp32 --steps 50 --precision fp32
run cavity100 --workload cavity100 --steps 50
run cavity100_fp32 --workload cavity100 --steps 50 --precision fp32
run cavity1000 --workload cavity1000 --steps 50
run shear --workload shear --steps 50
run shear_fp32 --workload shear --steps 50 --precision fp32
run tgv_config1 --workload tgv --steps 200
run duct_config2 --workload duct --steps 200
run strong_1gpu --workload strong --steps 20
run weak_aa --steps 50 --streaming aa
run weak_aa_fp32 --steps 50 --streaming aa --precision fp32
run cavity_aa --workload cavity100 --steps 50 --streaming aa
run weak_rm --steps 50 --model rm
run weak_fd --steps 30 --corrections full_fd
run weak_fd_fp32 --steps 30 --corrections full_fd --precision fp32
LBM_FD_TMA=0 run weak_fd_twopass --steps 30 --corrections full_fd
run cavity_fd --workload cavity100 --steps 50 --corrections full_fd
run weak_fd_lag --steps 50 --corrections full_fd_lag
run weak_fd_lag_fp32 --steps 50 --corrections full_fd_lag --precision fp32
run weak_halo_nccl --steps 50 --halo nccl
run weak_halo_p2p --steps 50 --halo p2p
run weak_fd_p2p --steps 30 --corrections full_fd --halo p2p
run weak_fp64_soak --steps 1000
run weak_fp32_soak --steps 1000 --precision fp32
