for rep in 1 2; do
python tools/time_main.py 3,4,6
for v in k4_fr1 h1_fr0 h1_fr2; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 4; done
for v in h1_k3_fr0 h1_k3_fr2; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 3; done
for v in h1_k6_fr1 h1_k6_fr3; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_main.py 6; done
done > gpurun_out/s6_ab_h1.jsonl 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_timeloop.py tests/test_gpu_curved.py -x -q > gpurun_out/s6_parity_h1.log 2>&1; tail -3 gpurun_out/s6_parity_h1.log
