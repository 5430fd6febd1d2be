for rep in 1 2; do
python tools/time_apply.py --k 4 --reps 40
for v in prep5 prep6 prepcp prepcp5; do echo "\"$v\""; HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_apply.py --k 4 --reps 40; done
done > gpurun_out/s6_ab_prep.jsonl 2>&1
