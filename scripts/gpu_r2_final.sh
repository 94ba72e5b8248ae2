# round-2 evidence run: smoke, full GPU suite, bench (headline + reference arm)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2f_host.txt; nproc >> gpurun_out/r2f_host.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2f_smoke.log
IGP_PARITY_LOG=gpurun_out/r2f_parity.json timeout 2700 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2f_pytest.log
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err; echo "bench ref rc $?"
