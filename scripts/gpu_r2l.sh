cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py tests/test_gpu_singular_aa_lid.py -k "aa or AA or streaming or wide or full_config3" -m gpu -q -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2l_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $1; }
run() { n=$1; shift; timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/r2l_$n.log 2>&1; echo "$n [$*]: $(summ gpurun_out/r2l_$n.log)"; }
run cavity_aa --workload cavity100 --steps 50 --streaming aa
run cavity_ab --workload cavity100 --steps 50
run weak_aa --steps 50 --streaming aa
run cavity_aa_fp32 --workload cavity100 --steps 50 --streaming aa --precision fp32
run shear_aa --workload shear --steps 20 --streaming aa
