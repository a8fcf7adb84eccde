# A/B of the chirp-z kernels at config 4 (default build vs paper_2602_17494_b200/libtvs_ab0.so)
set -x
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_full_size.py::test_config4_step1_first_sweep_sampled tests/test_gpu_golden.py::test_config4_short_schedule_full_size > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
for i in 1 2; do
timeout 300 python tools/c4_step1_short.py 8 > gpurun_out/ab_new_$i.json 2>gpurun_out/ab_new.err; echo "new rc=$?"
TVS_LIB_PATH=$PWD/paper_2602_17494_b200/libtvs_ab0.so timeout 300 python tools/c4_step1_short.py 8 > gpurun_out/ab_old_$i.json 2>gpurun_out/ab_old.err; echo "old rc=$?"
done
cat gpurun_out/ab_new_2.json gpurun_out/ab_old_2.json
