# Per-config bench lines (current kernels) into gpurun_out/configs/, then the
# DAS GPU tests.  Run under gpurun after the build.
set -u
mkdir -p gpurun_out/configs
b() { name=$1; shift; timeout 600 python bench.py --no-cpu "$@" > gpurun_out/configs/$name.log 2>&1
  tail -1 gpurun_out/configs/$name.log > gpurun_out/configs/bench_$name.jsonl
  echo "[$name] $(tail -1 gpurun_out/configs/$name.log | cut -c1-200)"; }
b cfg2 --steps 20
b cfg1 --config cfg1 --steps 20
b cfg3 --config cfg3 --frames 8 --steps 10 --no-e2e
b cfg5 --config cfg5 --steps 5
b cfg4 --frames 256 --steps 4 --no-e2e
b cfg2_nearest --interp nearest --steps 20 --no-e2e
b cfg1_nearest --config cfg1 --interp nearest --steps 20 --no-e2e

b sta_paper --config sta-paper --steps 10 --no-e2e
b sta_paper_nearest --config sta-paper --interp nearest --steps 10 --no-e2e
b pwi_paper --config pwi-paper --steps 20 --no-e2e
b cfg2_hann_f15 --window hann --f-number 1.5 --steps 20 --no-e2e
