timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
