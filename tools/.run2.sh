for rep in 1 2; do
python tools/time_main.py 3,4,5,6
for v in nosym_k4 k4_fr1 k4_fr3 k4_wreg; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 4; done
HDGC_LIB=tools/variants/nosym_k3/libhdgconv.so python tools/time_main.py 3
HDGC_LIB=tools/variants/nosym_k5/libhdgconv.so python tools/time_main.py 5
HDGC_LIB=tools/variants/nosym_k6/libhdgconv.so python tools/time_main.py 6
done > gpurun_out/s6_ab_sym.jsonl 2>&1
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s6_parity_sym.log 2>&1; tail -3 gpurun_out/s6_parity_sym.log
