set -x
python -c "import __graft_entry__ as g; g.build()"
for v in paper_2509_06220_b200/libnrmf.so build/variants/skip_nopf.so build/variants/noskip_pf.so build/variants/noskip_nopf.so; do echo "== $v"; python tools/c5_time.py $v; done > gpurun_out/r2c_c5.txt 2>&1
python tools/bench_variants.py paper_2509_06220_b200/libnrmf.so build/variants/noskip_nopf.so build/variants/skip_nopf.so build/variants/noskip_pf.so paper_2509_06220_b200/libnrmf.so build/variants/noskip_nopf.so > gpurun_out/r2c_variants.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_p2p.py tests/test_gpu_fastpath.py -x -q -p no:cacheprovider -k "not exhaustive" 2>&1 | tail -5 > gpurun_out/r2c_pytest.txt
