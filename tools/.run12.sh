for rep in 1 2; do
python tools/time_apply.py --k 4,5,6,7,8 --reps 30
for v in prep7 prep8; do echo "\"$v\""; HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_apply.py --k 4 --reps 30; done
for v in prepk5_4 prepk5_5; do echo "\"$v\""; HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_apply.py --k 5 --reps 30; done
for v in prepk6_4 prepk6_5; do echo "\"$v\""; HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time_apply.py --k 6 --reps 30; done
echo '"prepk7_3"'; HDGC_LIB=tools/variants/prepk7_3/libhdgconv.so python tools/time_apply.py --k 7 --reps 30
echo '"prepk8_3"'; HDGC_LIB=tools/variants/prepk8_3/libhdgconv.so python tools/time_apply.py --k 8 --reps 30
python tools/time3d.py 3
for v in prep3d_3 prep3d_4; do HDGC_LIB=tools/variants/$v/libhdgconv.so python tools/time3d.py 3; done
done > gpurun_out/s6_ab_prep2.jsonl 2>&1
