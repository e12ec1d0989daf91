cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/smp
for v in smp384 smp512; do PTUCKER_LIB=paper_1710_02261_b200/_variants/$v/libptucker.so timeout 120 python tools/quick_update.py c3 0.005 0 >> gpurun_out/smp/quick.txt 2>&1 || echo "fail $v" >> gpurun_out/smp/quick.txt; done
bash tools/ab_libs.sh c3 "prod smp384 smp512"
mv gpurun_out/ab.txt gpurun_out/smp/ab.txt
