python tools/ab.py build/variants/cur.so build/variants/l2n.so build/variants/l2l.so --rounds 5 > gpurun_out/r2q_ab.txt 2>&1
for v in build/variants/cur.so build/variants/l2n.so build/variants/l2l.so; do echo "== $v"; python tools/c5_time.py $v; done > gpurun_out/r2q_c5.txt 2>&1
