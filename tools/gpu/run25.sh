mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum"
for slot in a g; do for c in 0 1; do
ncu $M --clock-control none --cache-control none -k regex:spmv_dict -s 5 -c 1 --csv --log-file gpurun_out/ncu_dict_${slot}_c$c.csv python tools/spmv_one.py t_rtanis7_256x64 0 $slot --opt dict_rows=1 --opt dict_chunk=$c > gpurun_out/ncu_dict_${slot}_c$c.log 2>&1
done; done
tail -2 gpurun_out/ncu_dict_a_c1.log
