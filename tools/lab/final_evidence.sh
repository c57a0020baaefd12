#!/bin/bash
# end-of-round evidence: the LLaVA bench line, then the steady-state serving launch list
# (ncu gpu__time_duration per launch, launches 40000-48000 of a 400-request replay)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/final
timeout 2000 python bench.py > gpurun_out/final/llava.json 2> gpurun_out/final/llava.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 40000 --launch-count 8000 --csv --log-file gpurun_out/final/launches.csv python tools/profile_serving.py --requests 400 --rate 85 > gpurun_out/final/ncu.log 2>&1
