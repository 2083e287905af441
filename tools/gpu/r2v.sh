python tools/c1_ab.py build/variants/short.so build/variants/cur.so build/variants/pol.so > gpurun_out/r2v_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/short.so > gpurun_out/r2v_c1b.txt 2>&1
python tools/c1_ab.py build/variants/short.so > gpurun_out/r2v_c1c.txt 2>&1
python tools/c1_ab.py build/variants/cur.so > gpurun_out/r2v_c1d.txt 2>&1
