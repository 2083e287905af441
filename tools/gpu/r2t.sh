set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/r2t_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2t_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r2t_ncu_d.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2t_s -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so s 2 30 > gpurun_out/r2t_ncu_s.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_split_kernel -c 1 -o gpurun_out/r2t_c1 -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 20 > gpurun_out/r2t_ncu_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/r2t_ncu_l.log 2>&1
