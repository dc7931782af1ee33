#!/bin/bash
# drop-in e2e output pages: 4 KB (default, MADV_NOHUGEPAGE) vs 2 MB (SSE_OUT_ALLOC=thp) on N GPUs
# (SSE_OUT_ALLOC=thp was removed after this A/B: slower at N=1 and N=4, `profiles/r02_ab_out_pages_rejected.log`)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r2_ab_outalloc_n$N.log; : > $out
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag >> $out 2>&1
B="bench.py --gpus $N --steps 1 --warmup 3 --cpu-atoms 0 --no-check --pi-steps 0 --phase-device-steps 0 --e2e-steps 2 --e2e-warmup 1"
run() {
  if [ $N -gt 1 ]; then timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 $B
  else timeout 1200 python $B; fi
}
for rep in 1 2; do
  for mode in "" thp; do
    echo "mode=${mode:-4k}: $(SSE_OUT_ALLOC=$mode run 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']
print('value', round(d['value'],4), 'e2e', round(e['value'],4), 'steps', [round(x,3) for x in e['step_s']], 'pack', e['host_pack_ms'], 'unpack', e['host_unpack_ms'], 'bitwise', e['bitwise_equal_to_device_run'])")" >> $out
  done
done
cat $out
