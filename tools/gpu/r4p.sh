set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r4p_pytest.txt
tail -3 gpurun_out/r4p_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4p_smoke.txt 2>&1; echo smoke $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r4p_bench.json 2> gpurun_out/r4p_bench.err
tail -c 400 gpurun_out/r4p_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r4p_ref.json 2>&1; tail -c 600 gpurun_out/r4p_ref.json
