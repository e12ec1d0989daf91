CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain11.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_r02.csv $CMD > gpurun_out/ncu11a.log 2>&1
$CMD > gpurun_out/plain11b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_update_tc -s 3 -c 1 -o gpurun_out/prof_c5_r02 $CMD > gpurun_out/ncu11b.log 2>&1
