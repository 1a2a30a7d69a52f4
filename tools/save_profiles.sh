#!/usr/bin/env bash
# Copy one gpu_r02.sh run's evidence into profiles/ (tracked): ncu summaries
# of the config-5 spread / interpolation (+ per-instruction stall tables),
# the launch list, the bench line, and the traffic entry bench.py reports.
# usage: bash tools/save_profiles.sh <tag> <round-prefix, e.g. r02>
set -e
tag=$1; pre=${2:-r02}
mkdir -p profiles/${pre}_bench
for k in spread interp; do
  { python tools/ncu_summary.py gpurun_out/${tag}_$k.ncu-rep;
    echo; echo '## per-instruction stall samples (SASS, `tools/sass_stalls.py`)'; echo; echo '```';
    python tools/sass_stalls.py gpurun_out/${tag}_$k.ncu-rep "${k}_v[67]" 30; echo '```'; } > profiles/${pre}_c5_${k}_ncu.md
done
cp gpurun_out/${tag}_launches.csv profiles/${pre}_launches_c5.csv
tail -1 gpurun_out/${tag}_bench.json > profiles/${pre}_bench/default_c5.json
python - <<PY
import json
p = "profiles/traffic.json"
d = json.load(open(p))
d.pop("config5", None)
json.dump(d, open(p, "w"), indent=1)
PY
python tools/make_traffic.py config5=gpurun_out/${tag}_spread.ncu-rep > /dev/null
python tools/make_traffic.py config5=gpurun_out/${tag}_interp.ncu-rep > /dev/null
echo saved
