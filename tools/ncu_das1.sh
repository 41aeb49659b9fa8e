# ncu --set full of the one-frame cfg2 DAS launch (tools/das1_probe.py cfg2),
# after the probe itself has exited 0 without ncu
python tools/das1_probe.py cfg2 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:das_tma -s 3 -c 1 -o gpurun_out/prof_das1 python tools/das1_probe.py cfg2 > gpurun_out/ncu_das1.log 2>&1
tail -2 gpurun_out/ncu_das1.log
