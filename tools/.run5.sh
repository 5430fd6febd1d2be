for rep in 1 2; do
HDGC_ZIGZAG=1 python tools/time_main.py 3,4,5,6,8
HDGC_ZIGZAG=0 python tools/time_main.py 3,4,5,6,8
HDGC_ZIGZAG=1 python tools/time_apply.py --k 4,6
HDGC_ZIGZAG=0 python tools/time_apply.py --k 4,6
done > gpurun_out/s6_ab_zz.jsonl 2>&1
python bench.py > gpurun_out/s6_bench_zz.jsonl 2>gpurun_out/s6_bench_zz.err
python -m pytest tests/test_gpu_parity.py tests/test_gpu_timeloop.py tests/test_gpu_curved.py tests/test_gpu_guards.py -x -q > gpurun_out/s6_parity_zz.log 2>&1; tail -3 gpurun_out/s6_parity_zz.log
