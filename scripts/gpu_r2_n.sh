mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_birch.py -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2_pytest_n.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r2_pytest_n.log
timeout 1500 python tools/config_times.py tiny,medium,headline,headline_degree,streaming,large,large_degree,large_noreorder --json gpurun_out/r2_config_times.json > gpurun_out/r2_config_times.txt 2>&1; cat gpurun_out/r2_config_times.txt
timeout 1500 python tools/oracle_times.py tiny,medium,headline,streaming,large --json gpurun_out/r2_oracle_times.json > gpurun_out/r2_oracle_times.txt 2>&1; tail -6 gpurun_out/r2_oracle_times.txt
nproc; lscpu | grep "Model name"
