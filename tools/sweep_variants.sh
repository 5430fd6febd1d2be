for d in tools/variants/*/; do n=$(basename $d); k=$(echo $n | sed 's/^k\([0-9]\).*/\1/'); HDGC_LIB=$d/libhdgconv.so python tools/time_main.py $k 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try:
        d=json.loads(l); print('$n', d['k'], round(d['main_us'],2))
    except Exception: print('$n', l.strip()[:100])
"; done
