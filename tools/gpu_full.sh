#!/bin/bash
# Full measurement pass (round artefacts): gpu tests, smoke, default bench, reference arm, launch
# list, ncu --set full captures of every kernel family, the SURVEY §8(d) side configs (each line
# with roofline, cpu_baseline and e2e), the E5 per-iteration profile.
#   usage (under gpurun): bash tools/gpu_full.sh TAG [skip-tests]
TAG=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/tests_$TAG.txt
  cat gpurun_out/tests_$TAG.txt
fi
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err
head -c 600 gpurun_out/bench_full_$TAG.json; echo
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
tail -1 gpurun_out/bench_ref_$TAG.json | head -c 300; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
NCU="timeout 400 ncu --set full --clock-control none --import-source on"
$NCU -k regex:decode_hyb8 -s 2 -c 1 -o gpurun_out/prof_hyb_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
$NCU -k regex:sos_tc -s 3 -c 1 -o gpurun_out/prof_sos_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c2 --rule 0 --probes 1000000 --opt sos_bits=0 > /dev/null 2>&1
$NCU -k regex:sos_bits -s 3 -c 1 -o gpurun_out/prof_sosbits_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c2 --rule 0 --probes 1000000 > /dev/null 2>&1
$NCU -k regex:sos_tc -s 1 -c 1 -o gpurun_out/prof_sosc4_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c4 --rule 0 --probes 100000 > /dev/null 2>&1
$NCU -k regex:decode_l2t -s 1 -c 1 -o gpurun_out/prof_l2_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c4 --rule 2 --probes 1000000 > /dev/null 2>&1
$NCU -k regex:decode_smem -s 3 -c 1 -o gpurun_out/prof_smem_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c2 --rule 1 --probes 1000000 > /dev/null 2>&1
$NCU -k regex:store_priv -s 2 -c 1 -o gpurun_out/prof_store_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c5 > /dev/null 2>&1
# SURVEY §8(d) side configs: C2 M sweep x rules at 10^5 probes, C4 at 10^6, C1 (1-thread oracle), Scenario 2, C5
rm -f gpurun_out/bench_rules_$TAG.jsonl
for M in 5000 10000 15000 20000 25000 30000; do
  for R in 0 1 2; do
    timeout 400 python bench.py --steps 10 --config c2 --messages $M --rule $R --cpu-budget 6 --e2e-steps 2 >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
  done
done
for a in "--config c2 --rule 0 --probes 1000000" "--config c2 --rule 0 --probes 1000000 --opt sos_bits=0" "--config c2 --rule 2 --probes 10000000" "--config c4 --rule 0" "--config c4 --rule 1" "--config c4 --rule 2" "--config s2 --rule 2" "--config s2 --rule 1" "--config s2 --rule 0"; do
  timeout 600 python bench.py --steps 10 --cpu-budget 6 --e2e-steps 2 $a >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
done
for R in 0 1 2; do
  timeout 300 python bench.py --steps 10 --config c1 --rule $R --cpu-threads 1 --cpu-budget 6 --e2e-steps 2 >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
done
timeout 300 python bench.py --steps 10 --config c5 >> gpurun_out/bench_rules_$TAG.jsonl 2>/dev/null
timeout 600 python tools/motivation.py gpurun_out/motivation_$TAG.json > /dev/null 2>&1
wc -l gpurun_out/bench_rules_$TAG.jsonl
ls gpurun_out | grep $TAG
