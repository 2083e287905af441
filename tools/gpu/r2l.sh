set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2l_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2l_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r2l_ncu_d.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r2l_s -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so s 2 30 > gpurun_out/r2l_ncu_s.log 2>&1
