set -x
HDGC_MODAL=0 python tools/time_main.py 4 256
HDGC_MODAL=4 python tools/time_main.py 4 256
HDGC_MODAL=0 HDGC_SFM3=1 python tools/time_main.py 4 256
for v in wreg0_m7 wreg0_m6 m4 wreg0_m5; do HDGC_LIB=tools/variants/$v/libhdgconv.so HDGC_MODAL=4 python tools/time_main.py 4 256; done
for v in m4 wreg0_m5; do HDGC_LIB=tools/variants/$v/libhdgconv.so HDGC_MODAL=0 HDGC_SFM3=1 python tools/time_main.py 4 256; done
