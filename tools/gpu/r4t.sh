python tools/trace_probe.py build/variants/trace1.so 28 > gpurun_out/r4t_trace28.txt 2>&1
head -40 gpurun_out/r4t_trace28.txt
timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-extras > gpurun_out/r4t_c1.json 2>&1; tail -c 300 gpurun_out/r4t_c1.json | head -c 300; echo
python -c "
import json; d=json.loads(open('gpurun_out/r4t_c1.json').read().strip().splitlines()[-1]); print(d['ms_per_step']*1e3, d.get('us_per_step_by_difference'))"
