set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r2a_pytest.txt
tail -5 gpurun_out/r2a_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -c 600 gpurun_out/r2a_bench.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2a_bench_c1.json 2>&1
for p in 0 1; do NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2960$p bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r2a_bench_c1_dist$p.json 2>&1; done
