#!/bin/bash
# measured FP64 FMA peak with the SM clock sampled during the run
# -> gpurun_out/fp64_peak.json (copy to profiles/round2_fp64_peak.json)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/fp64_clocks.csv &
SMI=$!
sleep 0.5
/tmp/fp64_peak > gpurun_out/fp64_peak_raw.json
kill $SMI; wait $SMI 2>/dev/null
python - <<'PY'
import json
r = json.load(open("gpurun_out/fp64_peak_raw.json"))
rows = [l.split(",") for l in open("gpurun_out/fp64_clocks.csv") if l.strip()]
mhz = sorted(float(x[0]) for x in rows if float(x[2]) > 300)   # under load
mx = float(rows[0][1]) if rows else 1965.0
med = mhz[len(mhz) // 2] if mhz else float("nan")
r.update({"sm_mhz_median_under_load": med, "sm_max_mhz": mx, "samples_under_load": len(mhz),
          "reasons": sorted({x[3].strip() for x in rows}),
          "derived_peak_tflops_at_max_clock": 148 * 64 * 2 * mx * 1e6 / 1e12,
          "how": "16 independent DFMA chains x 256 threads x 8 CTAs/SM; burst = best of 5 launches, sustained = 4 s back to back; clocks from nvidia-smi every 100 ms"})
json.dump(r, open("gpurun_out/fp64_peak.json", "w"), indent=1)
print(json.dumps(r))
PY
