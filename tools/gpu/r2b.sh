set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_graph.py tests/test_gpu_p2p.py tests/test_gpu_dist_ranks.py -x -q -p no:cacheprovider -k "not exhaustive" 2>&1 | tail -15 > gpurun_out/r2b_pytest.txt
tail -3 gpurun_out/r2b_pytest.txt
python tools/c5_time.py > gpurun_out/r2b_c5_new.txt 2>&1
python tools/c5_time.py variants/exact.so > gpurun_out/r2b_c5_old.txt 2>&1
python tools/bench_variants.py paper_2509_06220_b200/libnrmf.so variants/exact.so paper_2509_06220_b200/libnrmf.so variants/exact.so > gpurun_out/r2b_variants.txt 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2b_bench_c1.json 2>&1
for p in 0 1; do NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2960$p bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2b_bench_c1_dist$p.json 2>&1; done
