#!/bin/bash
# GPU box: headline CSR (degree and planted order), then the register- vs shared-memory-index lab.
out=${1:-gpurun_out/smidx_lab.txt}
mkdir -p gpurun_out
[ -f /tmp/labd.ci ] || python tools/lab/prep_csr.py headline /tmp/labd > $out 2>&1
[ -f /tmp/labp.ci ] || python tools/lab/prep_csr.py headline /tmp/labp planted >> $out 2>&1
NNZ=$(python -c "import os;print(os.path.getsize('/tmp/labd.ci')//4)")
echo "== degree" >> $out; timeout 300 ./tools/lab/smidx_lab /tmp/labd.rp /tmp/labd.ci 1000000 $NNZ >> $out 2>&1
echo "== planted" >> $out; timeout 300 ./tools/lab/smidx_lab /tmp/labp.rp /tmp/labp.ci 1000000 $NNZ >> $out 2>&1
cat $out
