# Session 4: long-row fold partials in global memory (libigp_gfold.so) vs shared memory
# (libigp_smemfold.so), occupancy 2 / 3, interleaved on one box; then targeted GPU parity tests.
mkdir -p gpurun_out/s4; out=gpurun_out/s4/ab_fold.txt; rm -f $out
for i in 1 2 3; do for v in smemfold gfold; do
  cp paper_2508_19737_b200/libigp_$v.so paper_2508_19737_b200/libigp.so
  for cfg in headline medium; do
    timeout 200 python tools/embed_sweep.py $cfg ${W:-32} 2,3 2>/dev/null | grep "occ=" | sed "s/^/$v /" >> $out
  done
done; done
cp paper_2508_19737_b200/libigp_gfold.so paper_2508_19737_b200/libigp.so
cat $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "layer_ws or headline_parity or headline_dynamic or star_hub or medium_config or maximum_d or dims_and_ragged or ragged_tail or paper_settings_full" \
  > gpurun_out/s4/pytest_fold.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/s4/pytest_fold.log
