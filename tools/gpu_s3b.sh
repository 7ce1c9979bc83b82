mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "boundary or sos_bits or kernel_selection or hyb8 or fuzz or cycle or pair or options or smoke or symbols" 2>&1 | tail -3
python bench.py > gpurun_out/bench_c3_s3b.json 2> gpurun_out/bench_c3_s3b.err; python -c "import json;d=json.load(open('gpurun_out/bench_c3_s3b.json'));r=d['roofline'];print('C3', d['value'], r['decode_ms_per_launch'], r['frac'], r.get('onchip',{}).get('frac'), 'e2e', d['e2e']['value'], d['e2e']['state_bits']['value'])"
for o in "" "--opt sos_bits=0"; do for M in 5000 10000 15000; do python bench.py --config c2 --rule 0 --messages $M --probes 1000000 --no-cpu --no-e2e --steps 10 $o | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('SOS', '$M', '$o', r['kernel'], r['decode_ms_per_launch'])"; done; done
python bench.py --config c1 --rule 0 --no-cpu --no-e2e --steps 10 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('C1 SOS', r['kernel'], r['decode_ms_per_launch'])"
python bench.py --config c1 --rule 0 --no-cpu --no-e2e --steps 10 --opt sos_bits=0 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('C1 SOS', r['kernel'], r['decode_ms_per_launch'])"
REPS=2 STEPS=10 bash tools/ab.sh "--config c2 --rule 0 --probes 1000000"
