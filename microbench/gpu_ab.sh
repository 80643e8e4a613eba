cd /root/repo
python -m pytest tests -m gpu -x -q -k "dense or config1 or kernels_agree" > gpurun_out/t1.log 2>&1; tail -1 gpurun_out/t1.log
python bench.py --steps 10 > gpurun_out/bench_cls.json 2>gpurun_out/bench_cls.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_cls.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['prepass_ms_per_launch'], d['e2e']['ms_per_step'])
"
