for rep in 1 2; do
python tools/time_main.py 2,3,4,5,6
HDGC_LIB=tools/variants/k4_fr0/libhdgconv.so python tools/time_main.py 4
HDGC_LIB=tools/variants/k3_fr0/libhdgconv.so python tools/time_main.py 3
HDGC_LIB=tools/variants/k6_fr4/libhdgconv.so python tools/time_main.py 6
HDGC_LIB=tools/variants/k2_minb10/libhdgconv.so python tools/time_main.py 2
python tools/time_apply.py --k 4,5,6
python tools/time3d.py 3
done > gpurun_out/s6_ab_final.jsonl 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py -x -q 2>&1 | tail -2
