cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/init
PT_INIT_REPS=3 PTUCKER_DEBUG=1 timeout 300 python tools/init_time.py > gpurun_out/init/init3.txt 2>&1
PT_INIT_REPS=3 PTUCKER_LIB=paper_1710_02261_b200/_variants/trim/libptucker.so PTUCKER_DEBUG=1 timeout 300 python tools/init_time.py > gpurun_out/init/init3t.txt 2>&1
