#!/bin/bash
# PDL A/B on one B200: needs paper_2511_01633_b200/ab_nopdl.so.bin (libglmx.so built without the
# launch_pdl / pdl_wait change) and ab_pdl.so.bin (with it) next to the package; alternates them
# under the C2 bench, then runs the GPU suite and smoke on the PDL build.
mkdir -p gpurun_out
for i in 1 2 3; do
 for v in nopdl pdl; do
  cp paper_2511_01633_b200/ab_$v.so.bin paper_2511_01633_b200/libglmx.so
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_${v}_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$i.json').read().strip().splitlines()[-1]);print('$v',$i,round(d['value']),round(d['e2e']['value']),round(d['raw_computed_tokens_per_s']),d['clocks']['sm_mhz'],d['roofline']['elementwise_ms_per_step'],d['roofline']['attention_ms_per_step'],d['roofline']['append_ms_per_step'])"
 done
done
cp paper_2511_01633_b200/ab_pdl.so.bin paper_2511_01633_b200/libglmx.so
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_pdl.log 2>&1; tail -2 gpurun_out/pytest_pdl.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
