# Round-2 measurements behind profiles/r02/ (run under gpurun; each section is independent):
#   bash scripts/gpu_r2_measure.sh [sweep|dsmem|birch|stream|configs|ncu|large|tcpredict] ...
mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
for what in "$@"; do
case $what in
sweep)    # filter-step variants (the staged warp-batch kernel lived at commit 67f51ad: IGP_LAYER_KERNEL=ws)
  python tools/embed_sweep.py headline 32 2 "IGP_ALT_DIR=0;IGP_ALT_DIR=1" > gpurun_out/r2_sweep.txt 2>&1
  python tools/embed_sweep.py large 16,32,64 2 >> gpurun_out/r2_sweep.txt 2>&1 ;;
dsmem)    # DSMEM vs L2 random-row gathers
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lab/dsmem_lab tools/lab/dsmem_lab.cu && \
  ./tools/lab/dsmem_lab > gpurun_out/r2_dsmem_lab.txt 2>&1 ;;
birch)    # BIRCH fit / predict times at the headline embedding
  python tools/birch_times.py headline 1.0,0.5 --oracle-rows 100000 > gpurun_out/r2_birch_times.txt 2>&1 ;;
stream)   # the streaming config (10 stages) as a bench line
  python bench.py --config streaming --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_streaming.json 2>&1 ;;
configs)  # device times of every config, oracle rates on the host cores
  python tools/config_times.py tiny,medium,headline,headline_degree,streaming,large,large_degree,large_noreorder \
      --json gpurun_out/r2_config_times.json > gpurun_out/r2_config_times.txt 2>&1
  python tools/oracle_times.py tiny,medium,headline,streaming,large --json gpurun_out/r2_oracle_times.json \
      > gpurun_out/r2_oracle_times.txt 2>&1 ;;
ncu)      # launch list + one --set full capture of the filter step (bench command), BIRCH fit capture
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
  $CMD > gpurun_out/r2_plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2_launches.csv $CMD \
      > gpurun_out/r2_ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 10 -c 1 -o gpurun_out/r2_prof_layer -f \
      $CMD > gpurun_out/r2_ncu_layer.log 2>&1
  python tools/birch_profile.py headline 20000 > gpurun_out/r2_bplain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:birch_fit -c 1 -o gpurun_out/r2_prof_birch -f \
      python tools/birch_profile.py headline 20000 > gpurun_out/r2_ncu_birch.log 2>&1 ;;
large)    # the Large config as a bench line + one --set full capture of its filter step (traffic)
  python bench.py --config large --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-birch \
      > gpurun_out/r2_bench_large.json 2> gpurun_out/r2_bench_large.err
  CMD="python tools/ncu_embed.py large 4"
  $CMD > gpurun_out/r2_plain_large.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 2 -c 1 -o gpurun_out/r2_prof_large -f \
      $CMD > gpurun_out/r2_ncu_large.log 2>&1 ;;
tcpredict)  # BIRCH predict: tensor-core path vs fp64 path at the streaming leg's scale, + ncu of the tc kernel
  python tools/birch_predict_bench.py 150000 200000 64 0.05 > gpurun_out/r2_tc_predict.txt 2>&1
  python tools/birch_predict_bench.py 20000 1000000 64 1.0 >> gpurun_out/r2_tc_predict.txt 2>&1
  python tools/birch_predict_bench.py 40000 200000 32 0.03 >> gpurun_out/r2_tc_predict.txt 2>&1
  CMD="python tools/birch_predict_bench.py 150000 200000 64 0.05 --profile"
  $CMD > gpurun_out/r2_tc_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_tc_launches.csv $CMD \
      > gpurun_out/r2_tc_ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:birch_tc_kernel -c 1 -o gpurun_out/r2_prof_tc -f \
      $CMD > gpurun_out/r2_ncu_tc.log 2>&1 ;;
esac
done
