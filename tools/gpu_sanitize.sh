#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py (every kernel family).
TAG=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/sanitizer_${tool}_$TAG.txt 2>&1
  tail -2 gpurun_out/sanitizer_${tool}_$TAG.txt
done
