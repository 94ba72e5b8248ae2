#!/bin/bash
# GPU box: headline CSR in planted-block order (~ the community order), then the store lab (+ ncu L2 counters).
out=${1:-gpurun_out/store_lab.txt}
mkdir -p gpurun_out "$(dirname "$out")"
[ -f /tmp/labp.ci ] || python tools/lab/prep_csr.py headline /tmp/labp planted > $out 2>&1
NNZ=$(python -c "import os;print(os.path.getsize('/tmp/labp.ci')//4)")
echo "== planted" >> $out; timeout 120 ./tools/lab/store_lab /tmp/labp.rp /tmp/labp.ci 1000000 $NNZ >> $out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --launch-skip 0 --launch-count 168 --csv ./tools/lab/store_lab /tmp/labp.rp /tmp/labp.ci 1000000 $NNZ \
  > gpurun_out/store_lab_ncu.csv 2>&1
cat $out
