cd /root/repo
for cfg in "16 4" "24 4" "32 4" "20 3"; do
  set -- $cfg
  SKC_BUILD_QSMS=$1 SKC_BUILD_K=$2 python bench.py --steps 10 > gpurun_out/e2e_$1_$2.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/e2e_$1_$2.json').read().strip().splitlines()[-1]); print('qsms $1 K $2', d['e2e']['ms_per_step'], d['e2e']['ms_per_step_median'], d['ms_per_step'])
"
done
