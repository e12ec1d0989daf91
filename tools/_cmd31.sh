PT_TRACE_CFG=c3 PT_TRACE_MODE=2 PTUCKER_LIB=paper_1710_02261_b200/_variants/trk/libptucker.so timeout 300 python tools/trace_tc.py 1.0 1 > gpurun_out/trace_c3m2.txt 2>&1
