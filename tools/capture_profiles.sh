#!/bin/bash
# usage (GPU box, from the repo root): tools/capture_profiles.sh <tag>
# One cfg5 step under `ncu --set full` (both launches), summarised on the box (the report
# with sources is larger than gpurun_out may carry), traffic.json refreshed and stamped,
# the launch list of a short bench run, and the bench lines of both arms.
# Everything lands in gpurun_out/<tag>_*; copy what should be judged into profiles/.
tag=${1:-r02b}
export MB4_SKIP_BUILD=1
rep=/tmp/${tag}_split_cfg5
python bench.py --steps 100 --warmup 5 > gpurun_out/${tag}_bench_cfg5.json 2> gpurun_out/${tag}_bench_cfg5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_reference_arm_cfg5.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:mb4_step3 -s 6 -c 2 -f -o $rep \
    python bench.py --profile-only --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
python tools/ncu_summary.py $rep.ncu-rep > gpurun_out/${tag}_split_cfg5.txt 2>&1
mkdir -p profiles
cp gpurun_out/${tag}_split_cfg5.txt profiles/${tag}_split_cfg5.txt
python tools/update_traffic.py $rep.ncu-rep profiles/${tag}_split_cfg5.txt > gpurun_out/${tag}_traffic_entry.json 2>&1
cp profiles/traffic.json gpurun_out/${tag}_traffic.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_cfg5.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_launches.log 2>&1
# second bench line after the captures: traffic.json now matches the kernel sources
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg5_with_traffic.json 2>/dev/null
tail -2 gpurun_out/${tag}_ncu.log
head -c 600 gpurun_out/${tag}_bench_cfg5.json; echo
