#!/bin/bash
# Round measurement: bench (N=1), then the ncu launch list and one --set full capture of
# the filter step, each after the same command has exited 0 without ncu.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
cat gpurun_out/bench_ref.json
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 40 -c 1 -o gpurun_out/prof_round -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc $?"
