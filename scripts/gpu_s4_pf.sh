# Session 4 experiment: L2 bulk prefetch of the next row batch's far first-chunk neighbours
# (IGP_PF_DIST = row distance threshold, 0 = off), interleaved on one box.
mkdir -p gpurun_out/s4; out=gpurun_out/s4/ab_pf.txt; rm -f $out
for i in 1 2 3; do
  for pf in 0 4096 16384 1; do
    echo "== pf $pf" >> $out
    timeout 200 python tools/embed_sweep.py headline 32 2 "IGP_PF_DIST=$pf" 2>/dev/null | grep "occ=" >> $out
  done
done
cat $out
