#!/bin/bash
# Quick GPU check of a kernel change (run under gpurun): a parity subset, then the cfg5 / cfg4
# bench lines without the e2e / CPU legs.  Output under gpurun_out/quick_<tag>.*
tag=${1:-q}
export MB4_SKIP_BUILD=1
timeout 480 python -m pytest -x -q tests/test_gpu_runs.py tests/test_gpu_parity.py ${QUICK_TESTS} \
    > gpurun_out/quick_${tag}.tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/quick_${tag}.tests.log
for c in cfg5 cfg4 cfg3; do
  timeout 120 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline \
      >> gpurun_out/quick_${tag}.bench.log 2>&1
done
tail -3 gpurun_out/quick_${tag}.tests.log
python - "$tag" <<'PY'
import json, sys
for l in open(f"gpurun_out/quick_{sys.argv[1]}.bench.log"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(d["config"]["workload"][:5], "value %.4g" % d["value"], "ms/step %.4f" % d["ms_per_step"],
              "kernel ms %.4f" % r["kernel_ms_per_step"], "by sweep", r.get("sweep_ms_by_index"),
              "sweeps/step", d.get("sweeps_per_step"), "frac %.3f" % r["frac"], "drift %.2g" % d["energy_drift"])
PY
