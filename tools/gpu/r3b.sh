set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_unaligned.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r3b_pytest.txt
tail -3 gpurun_out/r3b_pytest.txt
PYTHONPATH=. python tools/unal_time.py > gpurun_out/r3b_unal.txt 2>&1
PYTHONPATH=. python tools/unal_time.py --lg 26 >> gpurun_out/r3b_unal.txt 2>&1
cat gpurun_out/r3b_unal.txt
true
tail -4 gpurun_out/r3b_ab.txt
