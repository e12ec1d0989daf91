CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain21.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_update_smp2 -s 2 -c 1 -o gpurun_out/prof_smp2_r02 $CMD > gpurun_out/ncu21.log 2>&1
PTUCKER_LIB=paper_1710_02261_b200/_variants/trk/libptucker.so timeout 300 python tools/trace_tc.py 1.0 1 1 > gpurun_out/trace_kcat.txt 2>&1
