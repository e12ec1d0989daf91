# usage: bash tools/trace_variant.sh "NVCC FLAGS" [policy]  -> gpurun_out/trace_variant.txt
cd $GRAFT_REPO_ROOT
touch paper_1710_02261_b200/csrc/update_tc.cu
NVCC_APPEND_FLAGS="-DPT_TRACE $1" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1
echo "== $1 policy=$2" >> gpurun_out/trace_variant.txt
PT_TRACE_POLICY=$2 python tools/trace_tc.py 1.0 >> gpurun_out/trace_variant.txt 2>&1
