cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2e2
for v in prod nobump prod nobump; do
  if [ $v = prod ]; then lib=""; else lib=paper_1710_02261_b200/_variants/$v/libptucker.so; fi
  echo "== $v" >> gpurun_out/e2e2/init.txt
  PTUCKER_LIB=$lib PT_INIT_REPS=4 timeout 300 python tools/init_time.py >> gpurun_out/e2e2/init.txt 2>&1
  PTUCKER_LIB=$lib python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench $v', d['e2e']['value'], d['e2e']['init_s'])" >> gpurun_out/e2e2/init.txt
done
