#!/bin/bash
# streaming stores into the pinned slots vs memcpy: the drop-in feed (bench e2e_dropin) and the feed probe, A/B/A/B
mkdir -p gpurun_out
for rep in 1 2; do for nt in 0 1; do
  DHSA_COPY_NT=$nt timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-records --no-probe > gpurun_out/nt${nt}_$rep.json 2> gpurun_out/nt${nt}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/nt${nt}_$rep.json')); print('nt=$nt', $rep, 'e2e', round(d['e2e']['value']), 'dropin', [(r['feeder_threads'], round(r['mpps'])) for r in d['e2e_dropin']['runs']])"
done; done
for nt in 0 1; do DHSA_COPY_NT=$nt timeout 600 python tools/host_feed_probe.py 2>&1 >/dev/null | grep workers | head -8 | sed "s/^/nt=$nt /"; done
