#!/bin/bash
export PYTHONPATH=.
for a in "4 64 17 17 1 7 0 3" "4 192 17 17 3 3 1 1" "4 192 17 17 1 7 0 3" "4 64 17 17 1 3 0 1" "4 128 17 17 1 7 0 3" "4 64 17 17 7 1 3 0" "4 64 17 17 3 5 1 2" "4 192 17 17 1 1 0 0"; do
  r=$(timeout 120 python scripts/i2c_probe.py $a 2>&1 | tail -1); echo "[$a] $r"
done
