set -x
python tools/ab.py build/variants/base.so build/variants/v_exact.so build/variants/noskip.so build/variants/v_safe1.so build/variants/v_safe2.so paper_2509_06220_b200/libnrmf.so --rounds 6 > gpurun_out/r2e_ab.txt 2>&1
for v in build/variants/v_safe1.so build/variants/v_safe2.so; do echo "== $v"; python tools/c5_time.py $v; done > gpurun_out/r2e_c5.txt 2>&1
