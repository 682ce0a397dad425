#!/bin/bash
# current tree vs the previous commit's build (tmp_prev/), same box
run() {
  (cd $1 && timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > /tmp/b.log 2>&1)
  python - "$2" <<'P'
import json,sys
l=json.loads(open('/tmp/b.log').read().strip().splitlines()[-1])
print(sys.argv[1], round(l['value']), round(l['ms_per_step'],3), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items()})
P
}
run $GRAFT_REPO_ROOT/tmp_prev prev
run $GRAFT_REPO_ROOT cur
run $GRAFT_REPO_ROOT/tmp_prev prev
run $GRAFT_REPO_ROOT cur
