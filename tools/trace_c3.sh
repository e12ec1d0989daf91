cd $GRAFT_REPO_ROOT
touch paper_1710_02261_b200/csrc/update_tc.cu
NVCC_APPEND_FLAGS="-DPT_TRACE" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1
PT_TRACE_CFG=c3 PT_TRACE_MODE=2 python tools/trace_tc.py 1.0 > gpurun_out/trace_c3.txt 2>&1
PT_TRACE_CFG=c5 PT_TRACE_MODE=1 python tools/trace_tc.py 0.1 >> gpurun_out/trace_c3.txt 2>&1
