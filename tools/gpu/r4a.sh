set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r4a_pytest.txt
tail -3 gpurun_out/r4a_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.txt 2>&1; echo smoke $?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
tail -c 400 gpurun_out/r4a_bench.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-extras > gpurun_out/r4a_bench_c1.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4a_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/r4a_ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r4a_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r4a_ncu_d.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_split_kernel -c 1 -o gpurun_out/r4a_c1 -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 20 > gpurun_out/r4a_ncu_c1.log 2>&1
