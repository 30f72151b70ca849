#!/bin/sh
# Round-end evidence on one B200 (run through gpurun from the repo root): bench lines for every
# BASELINE config, the ncu launch list and one `ncu --set full` capture of a training step, the
# cfg5 sweep.  Outputs under gpurun_out/$R/ (R = round tag, default r2).
R=${1:-r2}
O=gpurun_out/$R
mkdir -p $O
python bench.py > $O/bench_fwd_bwd_B8_L1024.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_reference_arm.json 2>> $O/bench.err
python bench.py --pass fwd --no-cpu-baseline > $O/bench_fwd_B8_L1024.json 2>> $O/bench.err
python bench.py --trunk 6 --B 4 --L 2048 --no-cpu-baseline > $O/bench_cfg3_trunk6_B4_L2048.json 2>> $O/bench.err
python bench.py --shard rows --B 1 --L 32768 --no-cpu-baseline > $O/bench_cfg4_rows_L32768.json 2>> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-attn-long > $O/launches_raw.csv 2>> $O/bench.err
FIPA_MICRO=1 ncu --set full --clock-control none --import-source on \
    -k regex:"attn_|gemm|proj_pack|bwd_|cast_inputs|recenter|finish" -c 20 -o $O/step_full \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-attn-long > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/step_full.ncu-rep \
    "FIPA_MICRO=1 ncu --set full --clock-control none --import-source on -k regex:\"attn_|gemm|proj_pack|bwd_|cast_inputs|recenter|finish\" -c 20 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-attn-long" \
    "B=8 L=1024 north-star shape, one fwd+bwd training step (first 20 matching launches)" > $O/step_ncu_summary.json
python tools/sweep.py --out $O/sweep.json > $O/sweep.log 2>&1
ls -la $O
