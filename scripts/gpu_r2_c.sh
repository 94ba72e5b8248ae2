mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python tools/embed_sweep.py headline 32 2 "IGP_LAYER_KERNEL=ws,IGP_WS_SHAPE=8x2;IGP_WS_SHAPE=4x4;IGP_WS_SHAPE=16x1;IGP_WS_SHAPE=6x2;IGP_LAYER_KERNEL=classic" > gpurun_out/r2_sweep4.txt 2>&1; cat gpurun_out/r2_sweep4.txt
IGP_QUICK=1 timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "not large and not maximum_csr and not paper_settings and not birch" > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/r2_pytest2.log
