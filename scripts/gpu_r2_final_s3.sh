# round-2 final evidence (session 3): smoke, full GPU suite (parity numbers), headline bench with
# in-run traffic (after the ncu capture is committed), launch list + ncu --set full of the
# headline filter step, reference arm.   bash scripts/gpu_r2_final_s3.sh [tests|ncu|bench|ref|large]
mkdir -p gpurun_out/s3f
for what in "$@"; do
case $what in
tests)
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3f/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/s3f/smoke.log
  IGP_PARITY_LOG=gpurun_out/s3f/parity.json timeout 2700 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider > gpurun_out/s3f/pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s3f/pytest.log ;;
ncu)
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
  $CMD > gpurun_out/s3f/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s3f/launches.csv $CMD \
      > gpurun_out/s3f/ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"layer_(ws_)?kernel" -s 10 -c 1 -o gpurun_out/s3f/prof_layer -f \
      $CMD > gpurun_out/s3f/ncu_layer.log 2>&1; echo "ncu rc $?" ;;
bench)
  timeout 900 python bench.py > gpurun_out/s3f/bench.json 2> gpurun_out/s3f/bench.err; echo "bench rc $?"; tail -1 gpurun_out/s3f/bench.json | cut -c1-300 ;;
ref)
  timeout 900 python bench.py --impl reference > gpurun_out/s3f/bench_ref.json 2> gpurun_out/s3f/bench_ref.err; echo "ref rc $?" ;;
large)
  timeout 900 python bench.py --config large --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-birch \
      > gpurun_out/s3f/bench_large.json 2> gpurun_out/s3f/bench_large.err; echo "large bench rc $?"
  CMD="python tools/ncu_embed.py large 4"
  $CMD > gpurun_out/s3f/plain_large.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"layer_(ws_)?kernel" -s 2 -c 1 -o gpurun_out/s3f/prof_large -f \
      $CMD > gpurun_out/s3f/ncu_large.log 2>&1; echo "ncu large rc $?" ;;
esac
done
