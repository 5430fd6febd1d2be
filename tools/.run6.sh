for rep in 1 2; do
python tools/time_main.py 4
for v in pf592 pf1184 pf2368; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 4; done
done > gpurun_out/s6_ab_pf.jsonl 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:conv2d_sf_kernel -c 12 --csv --log-file gpurun_out/s6_dram_instream_k4.csv python tools/prof_substep.py 4 > gpurun_out/s6_dram_instream.log 2>&1
