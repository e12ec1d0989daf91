cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/w2
ok=""
for v in wg3g6 wg3g8 wg3g8a6; do
  PTUCKER_LIB=paper_1710_02261_b200/_variants/$v/libptucker.so timeout 120 python tools/quick_update.py c5 0.001 0 >> gpurun_out/w2/quick.txt 2>&1 && ok="$ok $v" || echo "fail $v" >> gpurun_out/w2/quick.txt
done
bash tools/ab_libs.sh c5 "prod $ok"
mv gpurun_out/ab.txt gpurun_out/w2/ab.txt
