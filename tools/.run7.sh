ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:conv2d_sf_kernel -c 12 --csv --log-file gpurun_out/s6_dram_instream_k4.csv python tools/prof_substep.py 4 > gpurun_out/s6_dram_instream.log 2>&1
HDGC_ZIGZAG=0 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:conv2d_sf_kernel -c 12 --csv --log-file gpurun_out/s6_dram_instream_k4_nozz.csv python tools/prof_substep.py 4 > gpurun_out/s6_dram_instream2.log 2>&1
for rep in 1 2; do HDGC_ZIGZAG=1 python tools/time3d.py 3; HDGC_ZIGZAG=0 python tools/time3d.py 3; done > gpurun_out/s6_ab_zz3d.jsonl 2>&1
python -m pytest tests/test_gpu_3d.py -x -q 2>&1 | tail -2
