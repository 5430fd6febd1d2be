set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02g_gputests.log 2>&1; echo "tests rc=$?"
python bench.py > gpurun_out/r02g_bench.jsonl 2> gpurun_out/r02g_bench.err; echo "bench rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"
python tools/time3d.py 1,2,3,4 > gpurun_out/r02g_time3d.jsonl 2>&1
python tools/time_apply.py --3d > gpurun_out/r02g_apply3d.jsonl 2>&1
python tools/configs_report.py > gpurun_out/r02g_configs.jsonl 2> gpurun_out/r02g_configs.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02g_ncu_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:prep_tile2d_kernel -c 2 -f -o gpurun_out/r02g_prep_k4 python tools/prof_substep.py 4 > gpurun_out/r02g_ncu_p4.log 2>&1
$NCU -k regex:prep_tile3d_kernel -c 2 -f -o gpurun_out/r02g_prep3d_k3 python tools/time3d.py 3 > gpurun_out/r02g_ncu_p3d.log 2>&1
