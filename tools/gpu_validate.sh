# Round validation on one B200: full GPU suite, default bench line; with VAL_NCU=1 also the ncu
# launch list of one bench step and --set full captures of kernel (a') and of the local chirp-z
# forward / inverse launches of a config-4 inner update.  Outputs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$VAL_NOTEST" ]; then
TVS_PARITY_LOG=$PWD/gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
head -c 400 gpurun_out/bench.json
if [ -n "$VAL_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep1s -s 4 -c 1 -o gpurun_out/sweep1 python tools/c4_step1_short.py 2 > gpurun_out/ncu_sweep1.log 2>&1; echo "ncu sweep1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_czt -s 4 -c 2 -o gpurun_out/czt python tools/c4_step1_short.py 1 > gpurun_out/ncu_czt.log 2>&1; echo "ncu czt rc=$?"
fi
