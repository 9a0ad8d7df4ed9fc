#!/bin/bash
# bench.py's N > 1 code path on a one-GPU box: every rank on cuda:0, gloo rendezvous (DHSA_BENCH_SAME_DEVICE=1).
# Not a measurement: it checks slicing, barriers, the merges and the JSON line.
mkdir -p gpurun_out
export DHSA_BENCH_SAME_DEVICE=1
run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}"; }
run 2 29511 --steps 2 --warmup 3 --packets 20000000 --no-e2e > gpurun_out/mr_config2_p2p.json 2> gpurun_out/mr_config2_p2p.err
run 2 29512 --steps 2 --warmup 3 --packets 20000000 --no-e2e --merge allgather > gpurun_out/mr_config2_ag.json 2> gpurun_out/mr_config2_ag.err
run 2 29515 --steps 2 --warmup 3 --packets 20000000 --no-e2e --merge partition > gpurun_out/mr_config2_part.json 2> gpurun_out/mr_config2_part.err
run 4 29516 --steps 2 --warmup 3 --config 3 --window-packets 200000000 --merge partition > gpurun_out/mr_config3_part.json 2> gpurun_out/mr_config3_part.err
run 4 29513 --steps 2 --warmup 3 --config 3 --window-packets 200000000 > gpurun_out/mr_config3.json 2> gpurun_out/mr_config3.err
run 2 29514 --impl reference --steps 1 --warmup 0 --packets 20000000 > gpurun_out/mr_reference.json 2> gpurun_out/mr_reference.err
for f in mr_config2_p2p mr_config2_ag mr_config2_part mr_config3 mr_config3_part mr_reference; do
  python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
    print('$f', d.get('impl', 'ours'), 'n_gpus', d['n_gpus'], 'value', round(d['value']), d.get('scaling'), d.get('config', {}).get('merge'), d.get('parity'))
except Exception as e:
    print('$f FAILED', e); print(open('gpurun_out/$f.err').read()[-1500:])
PY
done
