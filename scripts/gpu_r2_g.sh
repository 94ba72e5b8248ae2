mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
IGP_PARITY_LOG=gpurun_out/r2_birch_parity.json timeout 1500 python -m pytest tests/test_gpu_birch.py -x -q --timeout 1200 -p no:cacheprovider > gpurun_out/r2_birch.log 2>&1; echo "pytest rc $?"; tail -30 gpurun_out/r2_birch.log; cat gpurun_out/r2_birch_parity.json
