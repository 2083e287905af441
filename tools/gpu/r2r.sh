set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/r2r_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.txt 2>&1
timeout 1500 python tools/fuzz_parity.py 1000 > gpurun_out/r2r_fuzz.txt 2>&1
timeout 2400 python tools/fuzz_parity.py 2000 --launch > gpurun_out/r2r_fuzz_launch.txt 2>&1
timeout 900 python tools/big_fp64_check.py > gpurun_out/r2r_big.txt 2>&1
