mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
export IGP_WS_SHAPE=10x2
python tools/ncu_embed.py headline 6 > gpurun_out/r2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:layer_ws -s 4 -c 1 -o gpurun_out/r2_prof_ws2 -f python tools/ncu_embed.py headline 6 > gpurun_out/r2_ncu.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/r2_ncu.log
