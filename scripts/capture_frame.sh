#!/bin/bash
# ncu evidence for one steady-state frame (GPU box): the launch list of the whole
# run, then a --set full capture of the launches of its last frame.
# Usage: bash scripts/capture_frame.sh TAG [WORKLOAD=C4] [WARM=30]
set -e
TAG=$1; W=${2:-C4}; WARM=${3:-30}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_all.csv \
    python scripts/profile_frame.py $W $WARM 1 8 > /dev/null
read SKIP COUNT < <(python - "$TAG" <<'PY'
import csv, sys
rows = [r for r in csv.reader(l for l in open(f"gpurun_out/{sys.argv[1]}_all.csv") if l.startswith('"'))]
h = rows[0]; k = h.index("Kernel Name"); i = h.index("ID")
names = [(int(r[i]), r[k]) for r in rows[1:]]
ing = [j for j, (_, n) in enumerate(names) if "k_ingest" in n]
print(names[ing[-1]][0], len(names) - ing[-1])
PY
)
python - "$TAG" "$SKIP" <<'PY'
import csv, sys
tag, skip = sys.argv[1], int(sys.argv[2])
lines = [l for l in open(f"gpurun_out/{tag}_all.csv") if l.startswith('"')]
rows = list(csv.reader(lines)); h = rows[0]; i = h.index("ID")
with open(f"gpurun_out/{tag}_launches.csv", "w") as f:
    f.write(lines[0])
    for l, r in zip(lines[1:], rows[1:]):
        if int(r[i]) >= skip:
            f.write(l)
PY
ncu --set full --clock-control none --import-source on --launch-skip $SKIP --launch-count $COUNT \
    -f -o gpurun_out/${TAG} python scripts/profile_frame.py $W $WARM 1 8 > /dev/null
echo "captured $COUNT launches from $SKIP"
