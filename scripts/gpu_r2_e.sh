mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
timeout 900 python tools/embed_sweep.py headline 32 2 "IGP_ALT_DIR=0;IGP_ALT_DIR=1;IGP_ALT_DIR=0;IGP_ALT_DIR=1" > gpurun_out/r2_altdir.txt 2>&1
timeout 1200 python tools/embed_sweep.py large 64 2 "IGP_ALT_DIR=0;IGP_ALT_DIR=1" >> gpurun_out/r2_altdir.txt 2>&1; cat gpurun_out/r2_altdir.txt
IGP_QUICK=1 timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "not large and not maximum_csr and not paper_settings and not birch" > gpurun_out/r2_pytest3.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_pytest3.log
