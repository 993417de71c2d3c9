#!/bin/bash
# e2e_ab.sh "G R L" ... : bench.py e2e (host pipeline) for groups G, ramp R, lookahead L
for gr in "$@"; do set -- $gr
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --other-configs 0 --like-for-like 0 --e2e-groups $1 --e2e-ramp $2 --e2e-lookahead $3 > gpurun_out/e2e_$1_$2_$3.json 2>gpurun_out/e2e.err
python -c "import json; d=json.load(open('gpurun_out/e2e_$1_$2_$3.json')); e=d['e2e']; print('$1 $2 $3', e['groups'], round(e['ms_per_step'],2), round(e['pcie_gbs'],1), round(d['ms_per_step'],2))" || tail -3 gpurun_out/e2e.err
done
