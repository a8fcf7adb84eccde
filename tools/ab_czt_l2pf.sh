# A/B of the chirp-z L2 prefetch at config 4 (default build vs paper_2602_17494_b200/libtvs_ab0.so),
# the czt parity tests and the bench-schedule energy test on the default build
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/ab_lib.sh 8 default libtvs_ab0.so
for f in gpurun_out/ab_*_2.json; do echo $f; python -c "
import json; d=json.load(open('$f')); print(d['seconds'], d['tau_hash'], d['families'].get('proj_fwd_czt'), d['families'].get('proj_inv_czt'))"; done
TVS_PARITY_LOG=$PWD/gpurun_out/parity_l2pf.jsonl timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_czt.py tests/test_gpu_golden.py::test_config4_short_schedule_full_size "tests/test_gpu_full_size.py::test_config4_bench_schedule_energies_oracle_evaluated" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
