#!/bin/bash
# C2 sweep (BASELINE configs[1]): 370M bf16 prefill, seq 2K-16K x batch 1-8, plus the C4 per-GPU
# point (2.7B, B=4, T=8192).  One bench line per point into gpurun_out/sweep_*.json.
set -u
for T in 2048 4096 8192 16384; do
  for B in 1 2 4 8; do
    timeout 300 python bench.py --model 370m --batch $B --seqlen $T --no-decode --no-cpu --no-c2 \
      --steps 5 --warmup 3 > gpurun_out/sweep_370m_B${B}_T${T}.json 2>/dev/null
  done
done
timeout 600 python bench.py --model 2.7b --batch 4 --seqlen 8192 --no-decode --no-cpu --no-c2 \
  --steps 5 --warmup 3 > gpurun_out/sweep_2p7b_B4_T8192.json 2>/dev/null
