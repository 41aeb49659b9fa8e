python tools/das1_probe.py 2>&1 | tail -8
ncu --set full --import-source on --clock-control none -k regex:das_tma -c 1 -o gpurun_out/prof_das1 python tools/das1_probe.py cfg2 > gpurun_out/ncu_das1.log 2>&1
tail -2 gpurun_out/ncu_das1.log
