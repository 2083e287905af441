set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r5d_pytest.txt
tail -3 gpurun_out/r5d_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5d_smoke.txt 2>&1; echo smoke $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r5d_bench.json 2> gpurun_out/r5d_bench.err
tail -c 300 gpurun_out/r5d_bench.err
