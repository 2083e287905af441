python tools/ab.py build/variants/cur.so build/variants/pair.so --rounds 6 > gpurun_out/r2p_ab.txt 2>&1
