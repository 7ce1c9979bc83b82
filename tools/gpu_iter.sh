#!/bin/bash
# One GPU iteration: parity tests, a short bench, one ncu --set full capture of the decode kernel.
# usage (under gpurun): bash tools/gpu_iter.sh TAG [bench args...]
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu --no-e2e "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));r=d['roofline'];print('value %.3e probes/s  decode %.3f ms  frac %.4f  kernel %s'%(d['value'],r['decode_ms_per_launch'],r['frac'],r['kernel']))"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
