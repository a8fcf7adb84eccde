# Round validation on one B200: full GPU suite, default bench line, the ncu launch list of a
# shortened bench step, one --set full capture of kernel (a').  Outputs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
head -c 400 gpurun_out/bench.json
if [ -n "$VAL_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep1s -s 4 -c 1 -o gpurun_out/sweep1 python tools/c4_step1_short.py 2 > gpurun_out/ncu_sweep1.log 2>&1; echo "ncu sweep1 rc=$?"
fi
