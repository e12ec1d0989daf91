timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64" > gpurun_out/t14.txt 2>&1
for c in "c5 --dtype f64" "c1" "c2" "c3" "c4" "c5"; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_all_r02.jsonl
done
