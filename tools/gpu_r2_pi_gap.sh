#!/bin/bash
# Pi wall time vs kernel time (host gaps) on the small and paper configs after caching the operand budget
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
for cfg in small paper; do
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0 > gpurun_out/r2_pigap_$cfg.log 2>&1
  grep '^{' gpurun_out/r2_pigap_$cfg.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); p=d['pi']; k=p['kernels']
print('$cfg', 'Pi wall', round(p['s_per_eval']*1e3,2), 'ms; kernels', round(sum(v['ms'] for v in k.values()),2), 'ms', {n: v['launches'] for n, v in k.items()})"
done
