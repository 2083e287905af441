set -x
python tools/trace2_probe.py build/variants/trace2.so 20 6 > gpurun_out/r3k_trace2.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/poll.so --rounds 5 > gpurun_out/r3k_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/poll.so --rounds 5 --dtype s >> gpurun_out/r3k_c1.txt 2>&1
for lg in 16 22; do python tools/c1_ab.py build/variants/cur.so build/variants/poll.so --rounds 3 --lg $lg >> gpurun_out/r3k_c1.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_split_ll.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r3k_pytest.txt
