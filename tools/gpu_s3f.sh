# re-measure the sum-of-sum lines that run sos_bits_kernel (C2 at 10^5 and 10^6 probes, C1) with the
# issue-slot on-chip figure; same arguments as tools/gpu_full.sh
mkdir -p gpurun_out; rm -f gpurun_out/bench_sosbits_s3f.jsonl
timeout 400 python bench.py --steps 10 --config c2 --messages 5000 --rule 0 --cpu-budget 6 --e2e-steps 2 >> gpurun_out/bench_sosbits_s3f.jsonl 2>/dev/null
timeout 600 python bench.py --steps 10 --cpu-budget 6 --e2e-steps 2 --config c2 --rule 0 --probes 1000000 >> gpurun_out/bench_sosbits_s3f.jsonl 2>/dev/null
timeout 300 python bench.py --steps 10 --config c1 --rule 0 --cpu-threads 1 --cpu-budget 6 --e2e-steps 2 >> gpurun_out/bench_sosbits_s3f.jsonl 2>/dev/null
wc -l gpurun_out/bench_sosbits_s3f.jsonl
