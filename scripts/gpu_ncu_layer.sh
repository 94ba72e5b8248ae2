# usage: bash scripts/gpu_ncu_layer.sh <config> <W> <occ> <tag>
mkdir -p gpurun_out
CMD="python tools/embed_sweep.py $1 $2 $3"
$CMD > gpurun_out/ncu_plain_$4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 20 -c 1 -o gpurun_out/prof_$4 -f $CMD > gpurun_out/ncu_$4.log 2>&1
echo "ncu rc $?"; tail -2 gpurun_out/ncu_$4.log
