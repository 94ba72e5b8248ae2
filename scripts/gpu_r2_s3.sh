# round-2 session-3 evidence: WS kernel tests, bench lines (headline, large), ncu captures of the
# filter-step kernels of both (traffic), launch list of the headline bench command
#   bash scripts/gpu_r2_s3.sh [tests|bench|ncu|large] ...
mkdir -p gpurun_out/s3
for what in "$@"; do
case $what in
tests)
  IGP_PARITY_LOG=gpurun_out/s3/parity_ws.json timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "layer_ws or large or headline" -p no:cacheprovider > gpurun_out/s3/pytest_ws.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3/pytest_ws.log ;;
bench)
  timeout 900 python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; echo "bench rc $?" ;;
ncu)
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
  $CMD > gpurun_out/s3/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s3/launches.csv $CMD \
      > gpurun_out/s3/ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"layer_(ws_)?kernel" -s 10 -c 1 -o gpurun_out/s3/prof_layer -f \
      $CMD > gpurun_out/s3/ncu_layer.log 2>&1; echo "ncu rc $?" ;;
large)
  timeout 900 python bench.py --config large --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-birch \
      > gpurun_out/s3/bench_large.json 2> gpurun_out/s3/bench_large.err; echo "large bench rc $?"
  CMD="python tools/ncu_embed.py large 4"
  $CMD > gpurun_out/s3/plain_large.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"layer_(ws_)?kernel" -s 2 -c 1 -o gpurun_out/s3/prof_large -f \
      $CMD > gpurun_out/s3/ncu_large.log 2>&1; echo "ncu large rc $?" ;;
esac
done
