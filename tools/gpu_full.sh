#!/bin/bash
# Full measurement pass (round artefacts): gpu tests, default bench, reference arm, launch list,
# ncu captures of the hybrid (C3), SOS (C2, C4), L2 (C4 hybrid) and store (C5) kernels, side configs.
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/tests_$TAG.txt
cat gpurun_out/tests_$TAG.txt
python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err
cat gpurun_out/bench_full_$TAG.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
tail -1 gpurun_out/bench_ref_$TAG.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
NCU="timeout 300 ncu --set full --clock-control none --import-source on"
$NCU -k regex:decode_hyb8 -s 2 -c 1 -o gpurun_out/prof_hyb_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
$NCU -k regex:sos_tc -s 3 -c 1 -o gpurun_out/prof_sos_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c2 --rule 0 --probes 1000000 > /dev/null 2>&1
$NCU -k regex:sos_tc -s 1 -c 1 -o gpurun_out/prof_sosc4_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --config c4 --rule 0 --probes 20000 > /dev/null 2>&1
$NCU -k regex:decode_l2t -s 1 -c 1 -o gpurun_out/prof_l2_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --config c4 --rule 2 --probes 1000000 > /dev/null 2>&1
$NCU -k regex:store_priv -s 2 -c 1 -o gpurun_out/prof_store_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c5 > /dev/null 2>&1
rm -f gpurun_out/bench_rules_$TAG.jsonl
for a in "--config c2 --rule 0" "--config c2 --rule 1" "--config c2 --rule 2" "--config c2 --rule 0 --probes 1000000" "--config c2 --rule 2 --probes 10000000" "--config c4 --rule 0 --probes 100000" "--config c4 --rule 1 --probes 100000" "--config c4 --rule 2" "--config c1 --rule 2" "--config s2 --rule 2" "--config s2 --rule 0" "--config c5"; do
  timeout 300 python bench.py --no-cpu --no-e2e --steps 10 $a >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
done
GB_SOS_FP4=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --config c2 --rule 0 --probes 1000000 >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
ls gpurun_out | tail -20
