# Round evidence: default bench line, the ncu launch list of the same command,
# and one ncu --set full capture of the DAS kernel (run after the plain bench
# has exited 0).
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1
python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:das_tma -c 1 \
    -o gpurun_out/prof_das_tma python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/bench_default.log
