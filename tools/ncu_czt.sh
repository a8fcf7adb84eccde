# ncu --set full of the two k_czt_r32 launches (forward, inverse) of one config-4 inner update
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_czt -s 2 -c 2 -o gpurun_out/czt_r32 python tools/c4_step1_short.py 1 > gpurun_out/ncu_czt.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_czt.log
