mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_birch.py -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2_pytest_i.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2_pytest_i.log
timeout 900 python tools/birch_times.py headline 1.0 > gpurun_out/r2_birch_times2.txt 2>&1; cat gpurun_out/r2_birch_times2.txt
