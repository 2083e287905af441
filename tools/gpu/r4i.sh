for lg in 10 12 14 16 18 20; do python tools/c1_ab.py build/variants/hdr.so --rounds 3 --lg $lg 2>&1 | grep median; done > gpurun_out/r4i_sizes.txt
cat gpurun_out/r4i_sizes.txt
