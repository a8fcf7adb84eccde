TVS_LIB_PATH=$PWD/paper_2602_17494_b200/libtvs_ph.so timeout 300 python tools/c4_step1_short.py 1 2>&1 | grep "czt kind" | sort | head -40 > gpurun_out/phases.txt
for i in 1 2; do
timeout 300 python tools/c4_step1_short.py 8 > gpurun_out/ab_new_$i.json 2>gpurun_out/ab_new.err; echo "new rc=$?"
done
timeout 300 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_golden.py::test_config4_short_schedule_full_size 2>&1 | tail -2
