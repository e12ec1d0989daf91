cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/nost
ok=""
for v in nost; do
  r=0
  for c in "c5 0.001 0" "c2 0.01 1" "c3 0.005 2"; do
    PTUCKER_LIB=paper_1710_02261_b200/_variants/$v/libptucker.so timeout 120 python tools/quick_update.py $c >> gpurun_out/nost/quick.txt 2>&1 || { echo "fail $v $c" >> gpurun_out/nost/quick.txt; r=1; }
  done
  [ $r = 0 ] && ok="$ok $v"
done
bash tools/ab_libs.sh c5 "prod $ok prod $ok"
bash tools/ab_libs.sh c3 "prod $ok"
mv gpurun_out/ab.txt gpurun_out/nost/ab.txt
