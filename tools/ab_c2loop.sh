# A/B of the F32-C2 order-5 kernel with the core in the constant bank read through the uniform
# datapath (pointer walk): variants c2l1 (levels 0 and 1 runtime loops), c2l2 (level 1 unrolled)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
bash tools/ab_libs.sh c4 "prod" 
bash tools/ab_libs.sh c4 "prod c2l1 c2l2" --policy F32-C2
for v in c2l1 c2l2; do
  PTUCKER_LIB=paper_1710_02261_b200/_variants/$v/libptucker.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -k "f32c2 or c4" 2>&1 | tail -4 >> gpurun_out/ab.txt
done
cat gpurun_out/ab.txt
