CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/prof_c4_r02 $CMD > gpurun_out/ncu29.log 2>&1
