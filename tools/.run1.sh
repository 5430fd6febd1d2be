set -x
python -m pytest tests -m gpu -x -q > gpurun_out/s6_gputests.log 2>&1; echo "tests rc=$?" 
python bench.py > gpurun_out/s6_bench.jsonl 2> gpurun_out/s6_bench.err; echo "bench rc=$?"
python tools/time_main.py 1,2,3,4,5,6,7,8 > gpurun_out/s6_time_main.jsonl 2>&1
python tools/time3d.py 1,2,3,4 > gpurun_out/s6_time3d.jsonl 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:conv2d_sf_kernel -c 3 -f -o gpurun_out/s6_sub_k4 python tools/prof_substep.py 4 > gpurun_out/s6_ncu_k4.log 2>&1
$NCU -k regex:conv2d_thread_kernel -c 3 -f -o gpurun_out/s6_sub_k2 python tools/prof_substep.py 2 > gpurun_out/s6_ncu_k2.log 2>&1
$NCU -k regex:prep_tile2d_kernel -c 2 -f -o gpurun_out/s6_prep_k4 python tools/prof_substep.py 4 > gpurun_out/s6_ncu_p4.log 2>&1
$NCU -k regex:conv3d_kernel -c 3 -f -o gpurun_out/s6_sub3d_k3 python tools/time3d.py 3 > gpurun_out/s6_ncu_3d.log 2>&1
$NCU -k regex:prep_tile3d_kernel -c 2 -f -o gpurun_out/s6_prep3d_k3 python tools/time3d.py 3 > gpurun_out/s6_ncu_p3d.log 2>&1
ls -la gpurun_out
