# full GPU suite + ncu of the tcgen05 router (8192 tokens, both shapes) + bench launch list
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/v_test.log)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:router -c 4 -o gpurun_out/router_tc_r02 -f python tools/ncu_router.py > gpurun_out/v_ncu_router.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 3 --serve-duration 0 --no-cpu-baseline > gpurun_out/v_ncu_bench.log 2>&1
timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/v_bench.log
