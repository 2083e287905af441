timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r4n_c1.json 2>&1
for p in 0 1; do NRMF_BENCH_DIST=1 NRMF_BENCH_P2P=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2960$p bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r4n_c1_dist$p.json 2>&1; done
timeout 900 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider 2>&1 | tail -3
for f in gpurun_out/r4n_c1*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step']*1e3, d.get('us_per_step_by_difference'), d.get('rank_exchange'), d.get('same_bits_as_1gpu_tree'))"; done
