M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
for lib in t3bk48 w_base w_kbig; do
  ATA_LIB_PATH=_ab/$lib.so ncu --metrics $M --clock-control none -k regex:prod_tf32 -c 1 --csv python tools/tf32_ab.py _ab/$lib.so > gpurun_out/ncu_$lib.csv 2>&1
done
