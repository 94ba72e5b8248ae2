mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
CMD="python bench.py --config streaming --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
$CMD > gpurun_out/r2_plain_stream.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_stream.csv $CMD > gpurun_out/r2_ncu_stream.log 2>&1
echo "ncu stream rc $?"
python tools/config_times.py streaming > gpurun_out/r2_ct_stream.txt 2>&1; tail -15 gpurun_out/r2_ct_stream.txt
