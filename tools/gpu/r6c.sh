set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r6c_d -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 30 > gpurun_out/r6c_ncu_d.log 2>&1; echo d $?
ncu --set full --import-source on --clock-control none -k regex:nrmf_split_kernel -c 1 -o gpurun_out/r6c_c1 -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so d 2 20 > gpurun_out/r6c_ncu_c1.log 2>&1; echo c1 $?
ncu --set full --import-source on --clock-control none -k regex:nrmf_tree_kernel -c 1 -o gpurun_out/r6c_s -f python tools/prof_one.py paper_2509_06220_b200/libnrmf.so s 2 30 > gpurun_out/r6c_ncu_s.log 2>&1; echo s $?
