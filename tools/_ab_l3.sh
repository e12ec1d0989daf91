cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.txt
bash tools/ab_libs.sh c4 "prod c2l3 prod c2l3"
PTUCKER_LIB=paper_1710_02261_b200/_variants/c2l3/libptucker.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "f32c2" 2>&1 | tail -n 3 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
