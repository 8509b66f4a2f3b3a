for r in 1 2; do for v in base ng8 ng8pu1 pu1; do LIB=variants/libpt_$v.so timeout 120 python tools/variant_time.py 2>&1 | tail -1; done; done
