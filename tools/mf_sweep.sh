#!/bin/bash
# usage: tools/mf_sweep.sh CONFIG STEPS "mf,m mf,m ..."   (run on the GPU box)
CFG=$1; STEPS=$2; shift 2
for pair in $1; do
  mf=${pair%,*}; m=${pair#*,}
  python bench.py --config $CFG --steps $STEPS --neumann $m --neumann-first $mf --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('$CFG mf=$mf m=$m', '%.3e'%d['value'], 'sweeps=%s'%d['sweeps_per_step'], 'drift=%.2e'%d['energy_drift'], 'frac=%.3f'%r['frac'], 'ms/step=%.3f'%r.get('kernel_ms_per_step', r['kernel_ms_per_launch']), r.get('sweep_ms_by_index'), (d['clocks'] or {}).get('sm_mhz'))"
done
