for pad in 0 8 1024; do python tools/trace_probe.py build/variants/trace.so 20 1 $pad; done > gpurun_out/r2y_trace.txt 2>&1
