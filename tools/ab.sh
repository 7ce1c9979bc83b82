#!/bin/bash
# Same-box A/B of library builds (run under gpurun).  Builds are compared inside ONE call: B200
# boxes differ by several percent, so numbers from different gpurun calls are not comparable.
#   local:  mkdir -p tools/ab && cp paper_1303_7032_b200/libgb.so tools/ab/libgb_old.so
#           (edit, rebuild) && cp paper_1303_7032_b200/libgb.so tools/ab/libgb_new.so
#   GPU:    gpurun -- 'bash tools/ab.sh "--config c3" "--config c2 --rule 2 --probes 10000000"'
# Prints decode ms per launch for every (repetition, build, config); variants are also
# selectable by environment knobs (GB_SOS_2CTA, GB_SOM_TC, ...) instead of builds.
REPS=${REPS:-2}
for rep in $(seq $REPS); do
  for lib in tools/ab/*.so; do
    for cfg in "$@"; do
      GB_LIB=$lib python bench.py $cfg --no-cpu --no-e2e --steps ${STEPS:-20} | \
        python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$(basename $lib)', '$cfg', r['decode_ms_per_launch'], d['ms_per_step'])"
    done
  done
done
