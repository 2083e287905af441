python tools/c1_ab.py build/variants/two.so build/variants/one.so --rounds 10 --reps 200 > gpurun_out/r5g_c1.txt 2>&1
python tools/c1_ab.py build/variants/two.so build/variants/one.so build/variants/two.so build/variants/one.so --rounds 6 --reps 200 >> gpurun_out/r5g_c1.txt 2>&1
for pad in 4 64 512; do python tools/c1_ab.py build/variants/one.so build/variants/two.so --rounds 4 --reps 200 --pad $pad >> gpurun_out/r5g_c1.txt 2>&1; done
grep median gpurun_out/r5g_c1.txt
