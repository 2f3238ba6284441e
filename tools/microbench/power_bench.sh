#!/usr/bin/env bash
# Run each power_bench mode for a few seconds while sampling SM clock / board power.
# Output: one line per mode with the op rate and the median clock / power of the last 2/3 of the run.
set -e
cd "$(dirname "$0")"
[ -x ./power_bench ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o power_bench power_bench.cu
SECS=${SECS:-4}
for mode in ${MODES:-dfma ffma int lds exp hbm}; do
  sleep 2
  nvidia-smi --query-gpu=clocks.sm,power.draw.instant --format=csv,noheader,nounits -lms 100 > /tmp/pw_$mode.csv &
  smi=$!
  res=$(./power_bench "$mode" "$SECS")
  kill $smi
  python3 - "$mode" "$res" <<'EOF'
import json, statistics, sys
mode, res = sys.argv[1], json.loads(sys.argv[2])
rows = [l.split(",") for l in open(f"/tmp/pw_{mode}.csv") if l.strip()]
rows = rows[len(rows) // 3:]
clk = statistics.median(float(r[0]) for r in rows)
pw = statistics.median(float(r[1]) for r in rows)
res.update({"sm_mhz": clk, "power_w": pw})
print(json.dumps(res))
EOF
done
