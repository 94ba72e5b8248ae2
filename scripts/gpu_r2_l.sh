mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "csr or stream or merge or adversarial or community or headline_csr" > gpurun_out/r2_pytest_l.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2_pytest_l.log

timeout 900 python bench.py --config streaming --steps 3 --warmup 3 --no-cpu-baseline --no-birch > gpurun_out/r2_bench_streaming2.json 2> gpurun_out/r2_bench_streaming2.err; echo "bench streaming rc $?"; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_streaming2.json'))
print([round(s['build_or_merge_ms'],3) for s in d['config']['stages']], d['config']['fresh_build_of_final_graph_ms'], d['config']['merge_stage9_vs_fresh_build'], d['value'])"
