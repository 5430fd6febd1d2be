for rep in 1 2; do
python tools/time3d.py 3
HDGC_LIB=tools/variants/nosym3d_k3/libhdgconv.so python tools/time3d.py 3
python tools/time_main.py 4,6
for v in ownf_fr0 ownf_fr1 ownf_fr2; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 4; done
for v in ownf_k3_fr0 ownf_k3_fr1; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 3; done
for v in ownf_k6_fr2 ownf_k6_fr3; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 6; done
done > gpurun_out/s6_ab_ownf.jsonl 2>&1
python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/s6_parity_3dsym.log 2>&1; tail -3 gpurun_out/s6_parity_3dsym.log
ncu --set full --clock-control none --import-source on -k regex:conv2d_sf_kernel -c 3 -f -o gpurun_out/s6b_sub_k4 python tools/prof_substep.py 4 > gpurun_out/s6b_ncu_k4.log 2>&1
