timeout 900 python tools/c4_policy_check.py 2,3 300 > gpurun_out/c4pol.txt 2>&1
for p in F32-C F32-C2; do timeout 300 python bench.py --config c4 --policy $p --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/c4bench.jsonl; done
