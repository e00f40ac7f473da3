#!/bin/bash
# A/B of the round-robin split's knobs on one GPU box (profiles/r02_lockstep_ab.txt):
# whole RK3 steps per variant with the defaults, the contiguous split
# (FDNS_ROUNDS=0), other unit sizes and the lockstep off, two interleaved rounds.
#   bash tools/ab_rounds.sh [size=512] [variants=SS,RS,SN]
set -u
SZ=${1:-512}; VS=${2:-SS,RS,SN}
run() { echo "== $*"; env "$@" python tools/step_timing.py --sizes "$SZ" --variants "$VS" --steps 6 2>&1 | grep "@"; }
for r in 1 2; do
  run X=default
  run FDNS_ROUNDS=0
  run FDNS_ROUNDS=64
  run FDNS_ROUNDS=256
  run FDNS_LOCKSTEP=0
  run FDNS_SS_FILL_PAIR=0
done
