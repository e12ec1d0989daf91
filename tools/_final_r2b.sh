cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fs2
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fs2/launches_bench_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fs2/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_update -s 6 -c 1 -o gpurun_out/fs2/c4_f32c2_full python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fs2/ncu_c4.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fs2/bench_ref.json 2> gpurun_out/fs2/bench_ref.err
rm -f gpurun_out/bench_all.jsonl gpurun_out/ab.txt; bash tools/ab_libs.sh c4 "prod mb3"; cp gpurun_out/ab.txt gpurun_out/fs2/ab_mb3.txt; bash tools/bench_all.sh > gpurun_out/fs2/bench_all.log 2>&1; cp gpurun_out/bench_all.jsonl gpurun_out/fs2/
ls -la gpurun_out/fs2
