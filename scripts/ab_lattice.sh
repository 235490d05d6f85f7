#!/bin/bash
# A/B of WC stage variants on one box (same build).  Each argument is one
# variant: a space-separated list of environment settings (default: the
# general pass-list kernel and the lattice kernel's forms).  Prints ms/step at 1.6h and 2h for each.
cd "$(dirname "$0")/.."
if [ $# -eq 0 ]; then
  set -- "SPHB_WC_LATTICE=0" "SPHB_LAT_UNIFORM_B=0" "SPHB_LAT_IB=0" "SPHB_LAT_MIRROR=0" "SPHB_LAT_MIRROR=1"
fi
for v in "$@"; do
  env $v python bench.py --steps 10 --warmup 3 --no-fp32 --no-c4 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || { echo "$v failed"; tail -5 /tmp/ab.err; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("/tmp/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], "|", d["roofline"]["kernel"], "1.6h %.3f ms/step (stage %.3f)" % (d["ms_per_step"], d["roofline"]["avg_launch_ms"]),
      "2h %.3f ms/step" % d["standard_2h"]["ms_per_step"], flush=True)
PY
done
