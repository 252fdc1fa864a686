#!/bin/bash
# helper back-off sweep on C2 (M=1) and random k'=3 N=128
for ns in 0 20 100; do
  echo "== DSGPU_HSLEEP=$ns"
  DSGPU_HSLEEP=$ns python tools/dbg_counters.py psi-mms 2 64 2>&1 | cut -c1-120
  DSGPU_HSLEEP=$ns DSGPU_REMOTE=4 python tools/dbg_counters.py random 3 128 2>&1 | cut -c1-120
done
