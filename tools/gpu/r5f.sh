cp build/variants/two.so paper_2509_06220_b200/libnrmf.so
timeout 1200 python -m pytest tests/test_gpu_split_ll.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_p2p.py tests/test_gpu_jitter.py tests/test_gpu_top_cr.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/c1_ab.py build/variants/one.so build/variants/two.so --rounds 10 --reps 200 > gpurun_out/r5f_c1.txt 2>&1
python tools/c1_ab.py build/variants/one.so build/variants/two.so --rounds 10 --reps 200 --dtype s >> gpurun_out/r5f_c1.txt 2>&1
python tools/c1_ab.py build/variants/one.so build/variants/two.so --rounds 6 --reps 200 --lg 21 >> gpurun_out/r5f_c1.txt 2>&1
grep median gpurun_out/r5f_c1.txt
