python tools/ab.py build/variants/cur.so build/variants/rul2.so build/variants/rul8.so --rounds 6 > gpurun_out/r2o_ab.txt 2>&1
