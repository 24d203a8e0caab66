#!/bin/bash
# Evidence for profiles/ (run on a B200 through gpurun, 1 GPU):
#   bench line, launch list of one C2 decode step, ncu --set full of the attention kernel and
#   the Tier-1 GEMMs of one layer (C2, batch 64) and of the large-batch pair kernel (batch 192).
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/cap
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err
python tools/engine_step.py --batch 64 --steps 1 --layers 2 --graph 0 > $O/step.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_raw.csv \
    python tools/engine_step.py --batch 64 --steps 1 --layers 2 --graph 0 > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_|gemm_tc|gemm_pair" -s 12 -c 6 \
    -o $O/full_c2 python tools/engine_step.py --batch 64 --steps 1 --layers 2 --graph 0 > $O/ncu_full.log 2>&1
python tools/engine_step.py --batch 192 --steps 1 --layers 2 --graph 0 > $O/step192.log 2>&1
ncu --set full --clock-control none -k regex:"gemm_pair|gemm_tc" -s 6 -c 5 \
    -o $O/full_b192 python tools/engine_step.py --batch 192 --steps 1 --layers 2 --graph 0 > $O/ncu_full192.log 2>&1
