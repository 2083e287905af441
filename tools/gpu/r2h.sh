set -x
python -c "import __graft_entry__ as g; g.build()"
python tools/trace_probe.py build/variants/trace.so 20 1 > gpurun_out/r2h_trace.txt 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2h_bench_c1.json 2>&1
NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2h_bench_c1_dist1.json 2>&1
timeout 900 python -m pytest tests/test_gpu_split_ll.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r2h_pytest.txt
