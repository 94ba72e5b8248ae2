mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
python tools/birch_profile.py headline 20000 > gpurun_out/r2_bplain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:birch_fit -c 1 -o gpurun_out/r2_prof_birch -f python tools/birch_profile.py headline 20000 > gpurun_out/r2_ncu_birch.log 2>&1
echo "ncu birch rc $?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
$CMD > gpurun_out/r2_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 10 -c 1 -o gpurun_out/r2_prof_layer -f $CMD > gpurun_out/r2_ncu_layer.log 2>&1
echo "ncu layer rc $?"; tail -2 gpurun_out/r2_ncu_layer.log
