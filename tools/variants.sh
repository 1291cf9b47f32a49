#!/bin/bash
# usage: tools/variants.sh "<bench args>" lib1.so lib2.so ...  (run on the GPU box)
ARGS="$1"; shift
for lib in "$@"; do
  MB4CU_LIB=$PWD/paper_2003_04345_b200/$lib python bench.py $ARGS --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('$lib', d['config']['workload'][:5], 'm=%s'%d['config']['neumann_terms'], '%.3e'%d['value'], d['sweeps_per_step'], 'frac=%.3f'%r['frac'], 'ms/step=%.3f'%r.get('kernel_ms_per_step', r['kernel_ms_per_launch']), r.get('sweep_ms_by_index'), (d['clocks'] or {}).get('sm_mhz'), 'drift=%.17g'%d['energy_drift'])"
done
