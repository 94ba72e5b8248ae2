mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
python tools/birch_profile.py headline 20000 > gpurun_out/r2_bplain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:birch_fit -c 1 -o gpurun_out/r2_prof_birch3 -f python tools/birch_profile.py headline 20000 > gpurun_out/r2_ncu_birch.log 2>&1
echo "ncu birch rc $?"
