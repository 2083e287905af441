set -x
timeout 1200 python -m pytest tests/test_gpu_split_ll.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_p2p.py tests/test_gpu_dist_ranks.py tests/test_gpu_top_cr.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r4h_pytest.txt
tail -3 gpurun_out/r4h_pytest.txt
python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so build/variants/lm.so --rounds 6 > gpurun_out/r4h_c1.txt 2>&1
python tools/c1_ab.py build/variants/cur.so build/variants/hdr.so build/variants/lm.so --rounds 6 --dtype s >> gpurun_out/r4h_c1.txt 2>&1
for lg in 16 22; do python tools/c1_ab.py build/variants/cur.so build/variants/lm.so --rounds 4 --lg $lg >> gpurun_out/r4h_c1.txt 2>&1; done
python tools/trace2_probe.py build/variants/trace2lm.so 20 6 > gpurun_out/r4h_trace2.txt 2>&1
grep median gpurun_out/r4h_c1.txt; head -20 gpurun_out/r4h_trace2.txt
