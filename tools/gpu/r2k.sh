python tools/ab.py build/variants/cur.so build/variants/pol.so build/variants/inc.so --rounds 8 > gpurun_out/r2k_ab.txt 2>&1
