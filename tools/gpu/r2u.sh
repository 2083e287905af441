python tools/c1_ab.py build/variants/pol.so build/variants/cur.so build/variants/short.so > gpurun_out/r2u_c1.txt 2>&1
python tools/c1_ab.py build/variants/pol.so build/variants/cur.so build/variants/short.so --lg 20 --dtype s >> gpurun_out/r2u_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/short.so build/variants/noshort.so --lg 28 --off 1 --flush 0 --reps 20 > gpurun_out/r2u_unal.txt 2>&1
