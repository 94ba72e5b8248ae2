# Interleaved A/B of whole bench steps (build + embed) on one box (tooling): prebuilt
# paper_2508_19737_b200/libigp_<name>.so variants alternate round by round.
#   bash scripts/ab_bench.sh <rounds> name...
rounds=$1; shift
mkdir -p gpurun_out/s3; out=gpurun_out/s3/ab_bench.txt; rm -f $out
cp paper_2508_19737_b200/libigp.so /tmp/libigp_default.so
for i in $(seq $rounds); do for v in "$@"; do
  cp paper_2508_19737_b200/libigp_$v.so paper_2508_19737_b200/libigp.so
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-birch 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('$v', round(d['value'],1), round(d['ms_per_step'],3), 'build', round(c['build_ms'],3), 'embed', round(c['embed_ms'],3), 'launch', round(d['roofline']['avg_launch_us'],1))" >> $out
done; done
cp /tmp/libigp_default.so paper_2508_19737_b200/libigp.so
cat $out
