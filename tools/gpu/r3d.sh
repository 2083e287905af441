set -x
python tools/c5_time.py build/variants/safe2.so > gpurun_out/r3d_c5.txt 2>&1
python tools/ab.py build/variants/head.so build/variants/safe2.so build/variants/sm0.so --rounds 8 > gpurun_out/r3d_ab.txt 2>&1
cat gpurun_out/r3d_c5.txt; tail -3 gpurun_out/r3d_ab.txt
