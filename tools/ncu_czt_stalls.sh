set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/c4_step1_short.py 2 > gpurun_out/short.json 2>gpurun_out/short.err; echo "short rc=$?"; cat gpurun_out/short.json | head -c 1500
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_czt -s 4 -c 2 -o gpurun_out/czt_r03 python tools/c4_step1_short.py 1 > gpurun_out/ncu_czt.log 2>&1; echo "ncu czt rc=$?"
tail -3 gpurun_out/ncu_czt.log
