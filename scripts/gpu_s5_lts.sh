# Session 5: the L2 slices' (LTS) own counters for one headline filter-step launch of the bench
# command -- how close the step is to the L2's throughput peak as ncu sees it.
mkdir -p gpurun_out/s5
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-birch"
M=gpu__time_duration.sum,lts__t_sectors.sum,lts__t_bytes.sum,lts__t_bytes.sum.per_second
M=$M,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.avg.pct_of_peak_sustained_elapsed
M=$M,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum
M=$M,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__cycles_elapsed.avg.per_second
M=$M,lts__cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_tag_requests.sum
M=$M,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,lts__d_sectors.avg.pct_of_peak_sustained_elapsed
M=$M,lts__xbar2lts_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_xbar2l1tex_read_sectors.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,dram__throughput.avg.pct_of_peak_sustained_elapsed
$CMD > gpurun_out/s5/lts_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:layer_kernel -s 20 -c 2 --csv --log-file gpurun_out/s5/lts_metrics.csv $CMD > gpurun_out/s5/lts_ncu.log 2>&1
echo "ncu rc $?"; tail -60 gpurun_out/s5/lts_metrics.csv | cut -c1-260
timeout 600 python bench.py > gpurun_out/s5/bench.json 2> gpurun_out/s5/bench.err; echo "bench rc $?"; cat gpurun_out/s5/bench.json
