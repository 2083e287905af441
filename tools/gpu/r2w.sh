for pad in 0 1 64 1024 4096; do python tools/c1_ab.py build/variants/short.so --pad $pad --rounds 3; done > gpurun_out/r2w_c1.txt 2>&1
python tools/c1_ab.py build/variants/short.so build/variants/short.so build/variants/short.so --rounds 3 >> gpurun_out/r2w_c1.txt 2>&1
python tools/c1_ab.py build/variants/short.so --wspad 2048 --rounds 3 >> gpurun_out/r2w_c1.txt 2>&1
