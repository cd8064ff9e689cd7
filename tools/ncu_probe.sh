python tools/trace_report.py
timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,gpu__time_duration.sum --clock-control none -k regex:decode_step -s 3 -c 1 python tools/perf_probe.py --ncu 2>&1 | grep -E "dram__|lts__|gpu__time" 
