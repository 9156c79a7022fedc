#!/bin/bash
# One GPU call's worth of round-end measurements (run under gpurun from the
# repo root): bench lines, configs, sweeps, the ncu launch list of the bench
# command and one `ncu --set full` capture of the step kernels.
#   bash tools/measure_round.sh TAG
set -u
TAG=${1:-rX}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --workload batch64 --no-cpu-baseline > $O/bench_batch64.json 2> $O/bench_batch64.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python tools/configs_bench.py > $O/configs.jsonl 2> $O/configs.err
python tools/size_sweep.py > $O/size_sweep.csv 2> $O/size_sweep.err
CHAN_SWEEP_TC_ONLY=1 python tools/chan_sweep.py 1000000 5 64:64 64:128 128:128 128:256 256:256 > $O/chan_sweep.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches_run.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_conv_(fwd|wgrad)_tc" -s 3 -c 3 \
  -o $O/full python tools/tc_perf.py 1000000 1 > $O/full_run.log 2>&1
ls -la $O
