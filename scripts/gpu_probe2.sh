#!/bin/bash
cd "$(dirname "$0")/.."
./scripts/green_probe 48 > gpurun_out/green.txt 2>&1
./scripts/green_probe 100 >> gpurun_out/green.txt 2>&1
FL_SOLO=0 FL_GROUPS=1 timeout 600 python scripts/wave_curve.py prof > gpurun_out/wave_prof.txt 2>&1
