set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python tools/fuzz_parity.py 5000 --seed=9101 > gpurun_out/r6b_fuzz.txt 2>&1; tail -1 gpurun_out/r6b_fuzz.txt
timeout 1200 python tools/fuzz_parity.py 3000 --launch --seed=9102 > gpurun_out/r6b_fuzz_launch.txt 2>&1; tail -1 gpurun_out/r6b_fuzz_launch.txt
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_jitter.py -q -p no:cacheprovider 2>&1 | tail -1; done > gpurun_out/r6b_jitter.txt
