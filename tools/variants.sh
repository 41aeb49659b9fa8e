timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.log 2>&1
tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms_per_frame'])"
timeout 300 python -m pytest tests/test_gpu_sigproc.py tests/test_gpu_pipeline.py -q 2>&1 | tail -2
