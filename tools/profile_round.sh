# Round evidence: GPU parity suite, smoke, the default bench line and the
# reference arm, the ncu launch list of the same bench command, and one
# ncu --set full capture per hot kernel (each after its plain run exited 0).
# ncu reports are summarised on the box (details page + raw csv) to keep
# gpurun_out small.
mkdir -p gpurun_out
summ() {  # $1 = report stem
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>&1
  gzip -f gpurun_out/$1_sass.csv
  rm -f gpurun_out/$1.ncu-rep
}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_gpu.log 2>&1; tail -2 gpurun_out/pt_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; tail -c 400 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; tail -c 300 gpurun_out/bench_reference.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai \
    > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:das_tma -s 3 -c 1 \
    -o gpurun_out/prof_das_tma python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai \
    > gpurun_out/ncu_das.log 2>&1; echo "das capture rc=$?"; summ prof_das_tma
timeout 600 ncu --set full --import-source on --clock-control none -k regex:analytic_reg -s 3 -c 1 \
    -o gpurun_out/prof_k2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai \
    > gpurun_out/ncu_k2.log 2>&1; echo "k2 capture rc=$?"; summ prof_k2
python tools/das1_probe.py > gpurun_out/das1.log 2>&1; tail -8 gpurun_out/das1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:das_tma -s 3 -c 1 \
    -o gpurun_out/prof_das1 python tools/das1_probe.py cfg2 no_json=1 > gpurun_out/ncu_das1.log 2>&1; echo "das1 capture rc=$?"; summ prof_das1
python tools/k2_probe.py > gpurun_out/k2.log 2>&1; tail -4 gpurun_out/k2.log
du -sh gpurun_out
