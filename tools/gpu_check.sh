# One GPU session: the parity suite, smoke, the default bench line and the
# reference arm (each log under gpurun_out/).
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pt_gpu.log 2>&1; tail -3 gpurun_out/pt_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -c 3000 gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; tail -c 1500 gpurun_out/bench_reference.log
