#!/bin/bash
# GPU-box check: parity tests, smoke, bench, and (optionally) ncu captures.
# usage: bash scripts/gpu_check.sh [tests] [bench] [ncu]
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv >> gpurun_out/host.txt
for what in "$@"; do
case $what in
tests)
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
  IGP_PARITY_LOG=gpurun_out/parity.json timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
  tail -15 gpurun_out/pytest_gpu.log ;;
bench)
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
  cat gpurun_out/bench.json ;;
ncu)
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 10 -c 1 -o gpurun_out/prof_layer -f $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc $?"; tail -3 gpurun_out/ncu_full.log ;;
esac
done
