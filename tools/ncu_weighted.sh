# ncu of the weighted (Hann, F = 1.5) cfg2 DAS launch, summarised on the box
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai --window hann --f-number 1.5 2>&1 | tail -1 | cut -c1-200
ncu --set full --import-source on --clock-control none -k regex:das_tma -s 3 -c 1 -o gpurun_out/prof_wt \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai --window hann --f-number 1.5 > gpurun_out/ncu_wt.log 2>&1
ncu -i gpurun_out/prof_wt.ncu-rep --page raw --csv > gpurun_out/prof_wt_raw.csv 2>&1
ncu -i gpurun_out/prof_wt.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_wt_sass.csv 2>&1
gzip -f gpurun_out/prof_wt_sass.csv; rm -f gpurun_out/prof_wt.ncu-rep
