set -x
python -c "import __graft_entry__ as g; g.build()"
python tools/ab.py paper_2509_06220_b200/libnrmf.so build/variants/noskip.so build/variants/base.so --rounds 6 > gpurun_out/r2d_ab.txt 2>&1
python tools/c5_time.py > gpurun_out/r2d_c5.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2d_pytest.txt
