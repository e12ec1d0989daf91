cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/w
for c in "c5 0.001 0" "c5 0.001 2" "c2 0.01 1" "c3 0.005 2" "c3 0.005 3"; do
  PTUCKER_LIB=paper_1710_02261_b200/_variants/wg3/libptucker.so timeout 120 python tools/quick_update.py $c >> gpurun_out/w/quick.txt 2>&1 || echo "fail $c rc=$?" >> gpurun_out/w/quick.txt
done
if ! grep -q fail gpurun_out/w/quick.txt; then
  bash tools/ab_libs.sh c5 "prod wg3"
  bash tools/ab_libs.sh c3 "prod wg3"
  mv gpurun_out/ab.txt gpurun_out/w/ab.txt
fi
