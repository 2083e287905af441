set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_split_ll.py tests/test_gpu_jitter.py tests/test_gpu_p2p.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2f_pytest.txt
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2f_bench_c1.json 2>&1
for p in 0 1; do NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2960$p bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2f_bench_c1_dist$p.json 2>&1; done
python tools/ab.py paper_2509_06220_b200/libnrmf.so build/variants/v_safe2.so build/variants/base.so --rounds 4 > gpurun_out/r2f_ab.txt 2>&1
python tools/c5_time.py > gpurun_out/r2f_c5.txt 2>&1
