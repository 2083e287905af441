set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r5b_pytest.txt
tail -3 gpurun_out/r5b_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5b_smoke.txt 2>&1; echo smoke $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r5b_bench.json 2> gpurun_out/r5b_bench.err
tail -c 300 gpurun_out/r5b_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5b_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/r5b_ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r5b_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r5b_ncu_d.log 2>&1
