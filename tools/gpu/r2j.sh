python tools/ab.py build/variants/cur.so build/variants/pol.so --rounds 8 > gpurun_out/r2j_ab.txt 2>&1
