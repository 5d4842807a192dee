# Two-process probe of C3's swap interference: process B copies pinned host ->
# device (or device -> host) in a loop in its own CUDA context while process A runs the C2-shape
# decode at batch 32 (128 GiB read per step) or 24 (96 GiB). First the event-timed slowdown
# without a profiler, then ncu counters of A's attention launches with B idle / busy (ncu
# serialises only A's own work; B's copy engines keep running).
# usage: bash tools/interference_ncu.sh   (outputs gpurun_out/intf_*)
python -m paper_2506_15155_b200.build > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_gcc.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_active.avg,l1tex__m_xbar2l1tex_read_sectors.sum,lts__t_requests_srcunit_tex.sum
bg() {  # kind seconds -> starts B, waits until it copies
  rm -f /tmp/intf_ready; python tools/h2d_loop.py --kind $1 --seconds $2 --ready /tmp/intf_ready > gpurun_out/intf_bg_$1_$3.log 2>&1 &
  BGPID=$!; for i in $(seq 120); do [ -f /tmp/intf_ready ] && break; sleep 1; done
}
for b in 32 24; do
  timeout 600 python tools/interference_probe.py --batch $b --label alone > gpurun_out/intf_t_${b}_alone.log 2>&1; tail -1 gpurun_out/intf_t_${b}_alone.log
  for kind in h2d d2h; do
    bg $kind 200 t$b
    timeout 600 python tools/interference_probe.py --batch $b --label $kind > gpurun_out/intf_t_${b}_$kind.log 2>&1; tail -1 gpurun_out/intf_t_${b}_$kind.log
    kill $BGPID; wait $BGPID 2>/dev/null; tail -1 gpurun_out/intf_bg_${kind}_t$b.log
  done
done
for b in 32 24; do
  timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -k regex:paged_attn -c 3 --csv \
    --log-file gpurun_out/intf_ncu_${b}_alone.csv python tools/interference_probe.py --batch $b --steps 1 --profiled 3 --label ncu_alone > gpurun_out/intf_ncu_${b}_alone.log 2>&1
  bg h2d 900 n$b
  timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -k regex:paged_attn -c 3 --csv \
    --log-file gpurun_out/intf_ncu_${b}_h2d.csv python tools/interference_probe.py --batch $b --steps 1 --profiled 3 --label ncu_h2d > gpurun_out/intf_ncu_${b}_h2d.log 2>&1
  kill $BGPID; wait $BGPID 2>/dev/null; tail -1 gpurun_out/intf_bg_h2d_n$b.log
done
ls gpurun_out/intf_*
