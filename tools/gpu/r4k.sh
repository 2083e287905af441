python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so build/variants/lm.so --rounds 8 --reps 200 > gpurun_out/r4k_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so build/variants/lm.so --rounds 8 --reps 200 --dtype s >> gpurun_out/r4k_c1.txt 2>&1
for lg in 16 22; do python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so build/variants/lm.so --rounds 5 --reps 200 --lg $lg >> gpurun_out/r4k_c1.txt 2>&1; done
grep median gpurun_out/r4k_c1.txt
