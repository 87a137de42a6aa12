#!/bin/bash
# Build stencil variants next to the production library (diagnostics):
#   tools/variants.sh R2C2G8 R1C2G16S3 ...  R = grid rows per lane, C = columns
#   per step, G = steps per chunk, S = ring slots (fast and exact)
cd "$(dirname "$0")/.."
for v in "$@"; do
  defs=$(python - "$v" <<'PY'
import re, sys
m = re.fullmatch(r"R(\d+)C(\d+)(?:G(\d+))?(?:S(\d+))?", sys.argv[1])
r, c, g, s = m.groups()
d = [f"-DSPTRSV_ST_R={r}", f"-DSPTRSV_ST_C={c}"]
if g: d.append(f"-DSPTRSV_ST_G={g}")
if s: d += [f"-DSPTRSV_ST_SLOTS_FAST={s}", f"-DSPTRSV_ST_SLOTS_EXACT={s}"]
print(" ".join(d))
PY
)
  python -m paper_2012_06959_b200.build --variant $v $defs > /dev/null &
done
wait
ls paper_2012_06959_b200/libsptrsv_b200_*.so
