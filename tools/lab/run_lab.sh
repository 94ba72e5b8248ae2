#!/bin/bash
# GPU box: prepare the headline CSR (degree and planted orders) and run the layer lab on both.
out=${1:-gpurun_out/lab.txt}
mkdir -p gpurun_out
[ -f /tmp/labd.ci ] || python tools/lab/prep_csr.py headline /tmp/labd > $out 2>&1
[ -f /tmp/labp.ci ] || python tools/lab/prep_csr.py headline /tmp/labp planted >> $out 2>&1
NNZ=$(python -c "import os;print(os.path.getsize('/tmp/labd.ci')//4)")
echo "== degree" >> $out; ./tools/lab/layer_lab /tmp/labd.rp /tmp/labd.ci 1000000 $NNZ >> $out 2>&1
echo "== planted" >> $out; ./tools/lab/layer_lab /tmp/labp.rp /tmp/labp.ci 1000000 $NNZ >> $out 2>&1
cat $out
