# full GPU check: tests, smoke, bench (default), ncu launch list + full capture of the tc kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rc
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/rc/tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rc/smoke.txt 2>&1
python bench.py > gpurun_out/rc/bench.json 2> gpurun_out/rc/bench.err
if [ "$1" = "ncu" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rc/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/rc/ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_update_tc -s 2 -c 1 -o gpurun_out/rc/tc_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/rc/ncu_full.log 2>&1
fi
