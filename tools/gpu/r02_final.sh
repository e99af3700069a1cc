# round-2 final validation: GPU suite, smoke, default bench, launch list of the bench command
(timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/f_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/f_test.log)
(timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/f_smoke.log)
(timeout 1200 python bench.py > gpurun_out/f_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/f_bench.log)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02e.csv python bench.py --steps 2 --warmup 3 --serve-duration 0 --no-cpu-baseline > gpurun_out/f_ncu_bench.log 2>&1
