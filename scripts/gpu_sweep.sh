mkdir -p gpurun_out
for c in ${4:-headline medium}; do python tools/embed_sweep.py $c ${1:-16,32,64} ${2:-2} "${3:-}"; done > gpurun_out/sweep.txt 2>&1
cat gpurun_out/sweep.txt
