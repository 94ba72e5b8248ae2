# Interleaved A/B of filter-step variants on one box (tooling): each variant is a prebuilt
# paper_2508_19737_b200/libigp_<name>.so and/or an env assignment; rounds alternate the variants
# so clock / power drift hits all of them alike.
#   bash scripts/ab_lib.sh <config> <rounds> "<name>[:ENV=V,...]" ...
cfg=$1; rounds=$2; shift 2
mkdir -p gpurun_out/s3; out=gpurun_out/s3/ab_${cfg}.txt; rm -f $out
cp paper_2508_19737_b200/libigp.so /tmp/libigp_default.so
for i in $(seq $rounds); do
  for v in "$@"; do
    name=${v%%:*}; env=""; [ "$name" != "$v" ] && env=${v#*:}
    if [ -f paper_2508_19737_b200/libigp_$name.so ]; then cp paper_2508_19737_b200/libigp_$name.so paper_2508_19737_b200/libigp.so
    else cp /tmp/libigp_default.so paper_2508_19737_b200/libigp.so; fi
    echo "== $v" >> $out
    timeout 300 python tools/embed_sweep.py $cfg ${W:-32} 2 "$env" >> $out 2>&1
  done
done
cp /tmp/libigp_default.so paper_2508_19737_b200/libigp.so
cat $out
