set -x
python -c "import __graft_entry__ as g; g.build()"
for ll in 1 0; do python tools/trace_probe.py build/variants/trace.so 20 $ll; done > gpurun_out/r2g_trace.txt 2>&1
