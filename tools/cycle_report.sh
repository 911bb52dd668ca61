#!/bin/bash
# Summarise one GPU cycle: launch shares, bench headline, ncu counters of the hot kernels.
TAG=$1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv 3 | tee profiles/${TAG}_launches.txt
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
d = json.loads(open('gpurun_out/bench_%s.json' % tag).read().strip().splitlines()[-1])
for k in ['value', 'ms_per_step', 'clocks', 'e2e', 'pass_ms_per_step', 'roofline']:
    print(k, json.dumps(d.get(k)))
PY
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > profiles/${TAG}_ncu_summary.json
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
b = json.loads(open('gpurun_out/bench_%s.json' % tag).read().strip().splitlines()[-1])
E = {'near_kernel': b['plan']['p2p_pairs'], 'p2p_kernel': b['plan']['p2p_pairs'], 'm2l_kernel': b['plan']['m2l_entries'], 'm2l_stored_kernel': b['plan']['m2l_entries']}
for d in json.load(open('profiles/%s_ncu_summary.json' % tag)):
    if d['kernel'] in E:
        e = E[d['kernel']]
        print(d['kernel'], 'ms %.3f' % d['time_ms'], 'fp64/entry %.1f' % ((d['dfma'] + d['dadd'] + d['dmul']) / e),
              'flops/entry %.1f' % ((2 * d['dfma'] + d['dadd'] + d['dmul']) / e),
              'inst/entry %.1f' % (d['warp_inst'] * 32 / e),
              'pipe %.1f issue %.1f warps %.1f regs %d' % (d['fp64_pipe_pct'], d['issue_pct'], d['warps_active_pct'], d['regs']))
PY
for k in m2l_stored p2p; do
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --kernel-name ${k}_kernel --launch-skip 0 --launch-count 1 2>/dev/null > gpurun_out/src_${k}_$TAG.csv
  echo "== $k"; python tools/stalls.py gpurun_out/src_${k}_$TAG.csv 6 | tee profiles/${TAG}_${k}_stalls.txt
done
if [ -f gpurun_out/prof_${TAG}_fly.ncu-rep ]; then
  python tools/ncu_summary.py gpurun_out/prof_${TAG}_fly.ncu-rep > profiles/${TAG}_fly_ncu_summary.json
  ncu -i gpurun_out/prof_${TAG}_fly.ncu-rep --page source --csv --kernel-name m2l_kernel --launch-skip 0 --launch-count 1 2>/dev/null > gpurun_out/src_m2l_$TAG.csv
  echo "== m2l (on the fly)"; python tools/stalls.py gpurun_out/src_m2l_$TAG.csv 6 | tee profiles/${TAG}_m2l_stalls.txt
fi
