#!/bin/bash
# ε sweep of the cfg5 populate (records committed / builds / wall) at a reduced then full resolution.
mkdir -p gpurun_out
for spec in "$@"; do
  timeout 600 python tools/populate_probe.py $spec 16384 >> gpurun_out/cfg5_probe.jsonl 2>> gpurun_out/cfg5_probe.err
  echo "done $spec rc=$?" >> gpurun_out/cfg5_probe.err
done
