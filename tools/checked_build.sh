# Bounds-checked build (compute-sanitizer is closed on this pool): PT_CHK asserts in the
# kernels (gathered-row coordinates and solved-row indices in range; a violation traps),
# loader role at 56 registers so the checks do not spill; then the GPU suite against it.
#   bash tools/checked_build.sh            (on the GPU box; the variant is built here first)
cd ${GRAFT_REPO_ROOT:-.}
[ -f paper_1710_02261_b200/_variants/checked/libptucker.so ] || \
  python -m paper_1710_02261_b200.build --variant checked -DPT_CHECKED -DPT_REG_P=56 -DPT_REG_L0=128
PTUCKER_LIB=paper_1710_02261_b200/_variants/checked/libptucker.so timeout 1500 \
  python -m pytest tests -m gpu -x -q -k "not fullsize_all" > gpurun_out/checked_suite.txt 2>&1
echo "rc=$?" >> gpurun_out/checked_suite.txt
