#!/bin/bash
# e2e (host-buffer) variance on one box: the probe + the bench's e2e leg (3 passes)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/e2evar2; mkdir -p $O
timeout 300 python tools/e2e_probe.py --steps 200 >> $O/probe.jsonl 2>> $O/probe.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench20.json 2> $O/bench20.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > $O/bench100.json 2> $O/bench100.err
timeout 300 python tools/e2e_probe.py --steps 200 >> $O/probe.jsonl 2>> $O/probe.err
cat $O/probe.jsonl
for f in $O/bench20.json $O/bench100.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"; done
