mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 1500 python tools/embed_sweep.py large 16,32,64 2 > gpurun_out/r2_large_w.txt 2>&1; cat gpurun_out/r2_large_w.txt
