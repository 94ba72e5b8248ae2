mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1

IGP_PARITY_LOG=gpurun_out/r2_parity_h.json timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "stream or merge or add_edges or community or birch or async" > gpurun_out/r2_pytest_h.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2_pytest_h.log

timeout 900 python tools/birch_times.py headline 1.0,0.5 --oracle-rows 100000 > gpurun_out/r2_birch_times.txt 2>&1; cat gpurun_out/r2_birch_times.txt
timeout 900 python bench.py --config streaming --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_streaming.json 2> gpurun_out/r2_bench_streaming.err; echo "bench streaming rc $?"; tail -c 1500 gpurun_out/r2_bench_streaming.json
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc $?"; tail -c 3000 gpurun_out/r2_bench.json
