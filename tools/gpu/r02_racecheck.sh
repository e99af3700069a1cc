# racecheck: minimal TMEM-alloc handoff repro (direct read vs relay), then the sanitize smoke over every path
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_race tools/scratch/tmem_alloc_race.cu
for v in 0 1; do timeout 300 compute-sanitizer --tool racecheck /tmp/tmem_race $v > gpurun_out/racecheck_repro_$v.log 2>&1; done
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_smoke.py > gpurun_out/racecheck_smoke.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/memcheck_smoke.log 2>&1
tail -n 3 gpurun_out/racecheck_repro_0.log gpurun_out/racecheck_repro_1.log gpurun_out/racecheck_smoke.log gpurun_out/memcheck_smoke.log
