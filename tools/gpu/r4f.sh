set -x
python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so --rounds 6 > gpurun_out/r4f_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so --rounds 6 --dtype s >> gpurun_out/r4f_c1.txt 2>&1
python tools/trace2_probe.py build/variants/trace2h.so 20 6 > gpurun_out/r4f_trace2.txt 2>&1
cat gpurun_out/r4f_c1.txt; head -20 gpurun_out/r4f_trace2.txt
