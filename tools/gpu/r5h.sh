set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r5h_pytest.txt
tail -3 gpurun_out/r5h_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5h_smoke.txt 2>&1; echo smoke $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r5h_bench.json 2> gpurun_out/r5h_bench.err
tail -c 300 gpurun_out/r5h_bench.err
python tools/trace2_probe.py build/variants/trace2two.so 20 6 > gpurun_out/r5h_trace2.txt 2>&1
for p in 1; do NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2962$p bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r5h_c1_dist$p.json 2>&1; done
