# usage: bash tools/trace_libs.sh "variant ..."  (variants built with -DPT_TRACE) -> gpurun_out/trace_libs.txt
cd $GRAFT_REPO_ROOT
for v in $1; do
  echo "== $v" >> gpurun_out/trace_libs.txt
  PTUCKER_LIB=paper_1710_02261_b200/_variants/$v/libptucker.so timeout 300 python tools/trace_tc.py 1.0 >> gpurun_out/trace_libs.txt 2>&1
done
