set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2i_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r2i_ncu_d.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2i_s -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so s 2 30 > gpurun_out/r2i_ncu_s.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_split_kernel -c 1 -o gpurun_out/r2i_c1 -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 20 > gpurun_out/r2i_ncu_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/r2i_ncu_l.log 2>&1
