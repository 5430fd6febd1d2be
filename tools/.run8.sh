for rep in 1 2; do
HDGC_TPREP=1 python tools/time_main.py 1,2
HDGC_TPREP=0 python tools/time_main.py 1,2
done > gpurun_out/s6_ab_tprep.jsonl 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/s6_gputests2.log 2>&1; tail -3 gpurun_out/s6_gputests2.log
