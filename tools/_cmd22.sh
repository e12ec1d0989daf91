timeout 120 env PTUCKER_LIB=paper_1710_02261_b200/_variants/nt4/libptucker.so python tools/quick_update.py c5 0.001 > gpurun_out/q22.txt 2>&1 || exit 1
bash tools/ab_libs.sh c5 "prod nt4"
PTUCKER_LIB=paper_1710_02261_b200/_variants/nt4t/libptucker.so timeout 300 python tools/trace_tc.py 1.0 1 1 > gpurun_out/trace_nt4.txt 2>&1
