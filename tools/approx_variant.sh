# usage: bash tools/approx_variant.sh "FLAGS" ... : rebuild approx.cu with FLAGS, time the scores (c5, c4 0.2)
cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/approx.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  echo "[$fl]" >> gpurun_out/sweep.txt
  python tools/time_scores.py c5 1.0 >> gpurun_out/sweep.txt 2>&1
  python tools/time_scores.py c4 0.2 >> gpurun_out/sweep.txt 2>&1
done
