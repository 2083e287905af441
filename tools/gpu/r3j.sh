set -x
python tools/trace2_probe.py build/variants/trace2.so 20 6 > gpurun_out/r3j_trace2.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/gpuscope.so --rounds 5 > gpurun_out/r3j_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/gpuscope.so --rounds 5 --dtype s >> gpurun_out/r3j_c1.txt 2>&1
cat gpurun_out/r3j_c1.txt
