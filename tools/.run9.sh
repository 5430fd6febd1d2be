set -x
python bench.py > gpurun_out/r02f_bench.jsonl 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02f_bench_ref.jsonl 2> gpurun_out/r02f_bench_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"
python tools/time_main.py 1,2,3,4,5,6,7,8 > gpurun_out/r02f_time_main.jsonl 2>&1
python tools/time3d.py 1,2,3,4 > gpurun_out/r02f_time3d.jsonl 2>&1
python tools/time_propagate.py > gpurun_out/r02f_propagate.jsonl 2>&1
python tools/time_richardson.py > gpurun_out/r02f_richardson.jsonl 2>&1
python tools/time_apply.py --k 4 > gpurun_out/r02f_apply.jsonl 2>&1
python tools/time_apply.py --3d >> gpurun_out/r02f_apply.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_ncu_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:conv2d_sf_kernel -c 3 -f -o gpurun_out/r02f_sub_k4 python tools/prof_substep.py 4 > gpurun_out/r02f_ncu_k4.log 2>&1
$NCU -k regex:conv2d_thread_kernel -c 3 -f -o gpurun_out/r02f_sub_k2 python tools/prof_substep.py 2 > gpurun_out/r02f_ncu_k2.log 2>&1
$NCU -k regex:conv2d_thread_kernel -c 3 -f -o gpurun_out/r02f_sub_k1 python tools/prof_substep.py 1 > gpurun_out/r02f_ncu_k1.log 2>&1
$NCU -k regex:conv3d_kernel -c 3 -f -o gpurun_out/r02f_sub3d_k3 python tools/time3d.py 3 > gpurun_out/r02f_ncu_3d.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:conv2d_sf_kernel -c 12 --csv --log-file gpurun_out/r02f_dram_instream_k4.csv python tools/prof_substep.py 4 > gpurun_out/r02f_dram_instream.log 2>&1
python tools/configs_report.py > gpurun_out/r02f_configs.jsonl 2> gpurun_out/r02f_configs.err
ls -la gpurun_out | tail -30
