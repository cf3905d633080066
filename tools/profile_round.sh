#!/bin/bash
# One-GPU evidence for profiles/: bench line, launch list, full ncu capture
# of the executor kernel (p=1 HBM copy and p=8 virtual all-reduce).
set -u
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench1.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python tools/profile_target.py ar1 > gpurun_out/pt_ar1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:persistent -s 2 -c 1 \
    -o gpurun_out/prof_ar1 python tools/profile_target.py ar1 > gpurun_out/ncu_ar1.log 2>&1
echo "ncu ar1 rc=$?"
python tools/profile_target.py ar8v --mib 256 > gpurun_out/pt_ar8v.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:persistent -s 2 -c 1 \
    -o gpurun_out/prof_ar8v python tools/profile_target.py ar8v --mib 256 > gpurun_out/ncu_ar8v.log 2>&1
echo "ncu ar8v rc=$?"
tail -1 gpurun_out/bench1.log
