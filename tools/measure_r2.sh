#!/bin/bash
# Round-2 measurements on the GPU box (outputs under gpurun_out/r2m_*):
# per-kernel step times, configs 1-4 (bf16 and the fp32 contract), the launch
# list of two bench steps, one ncu --set full capture of the forward and the
# fused backward.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 300 python tools/tc_perf.py 1000000 10 bf16 > $O/r2m_tcperf_bf16.txt 2>&1
timeout 300 python tools/tc_perf.py 1000000 5 f32tc > $O/r2m_tcperf_f32tc.txt 2>&1
timeout 900 python tools/configs_bench.py c1 c2 c3 c4 --math bf16 > $O/r2m_configs_bf16.jsonl 2> $O/r2m_configs.err
timeout 900 python tools/configs_bench.py c2 c3 c4 --math auto > $O/r2m_configs_auto.jsonl 2>> $O/r2m_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_conv|k_to_bf16|k_pack_w|k_wgrad_reduce" -s 14 -c 14 --csv \
  --log-file $O/r2m_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --fp32-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_(fwd_tc|bwd_fused)" -s 4 -c 2 \
  -o $O/r2m_full python tools/tc_perf.py 1000000 1 bf16 > $O/r2m_ncu.log 2>&1
echo measure done
