set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6a_smoke.txt 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r6a_pytest.txt
tail -3 gpurun_out/r6a_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r6a_bench.json 2> gpurun_out/r6a_bench.err
tail -c 300 gpurun_out/r6a_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6a_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/r6a_ncu_l.log 2>&1; echo ncu $?
