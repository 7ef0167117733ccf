#!/bin/bash
# Shared-memory wavefront and float64 rates on this B200 (tools/micro/peaks_smem_fp64.cu)
# -> profiles/peaks_smem.json, profiles/peaks_fp64.json (the roofline denominators
# bench.py uses for the forest walk and the exact float64 paths).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/peaks_smem_fp64 tools/micro/peaks_smem_fp64.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/peaks_clock.txt
./tools/micro/peaks_smem_fp64 > gpurun_out/peaks_smem_fp64.json || exit 1
python - <<'PY'
import json
d = json.load(open("gpurun_out/peaks_smem_fp64.json"))
clk = open("gpurun_out/peaks_clock.txt").read().strip()
common = {"gpu": d["gpu"], "sms": d["sms"], "how": "tools/micro/peaks_smem_fp64.cu: one 1024-thread CTA per SM, "
          "8 independent ops per thread per iteration, clock64() per CTA (median CTA)", "nvidia_smi_clocks": clk}
smem = dict(common, **{k: v for k, v in d.items() if k.startswith("smem_")})
smem["wavefronts_per_sm_clk"] = d["smem_lds32_conflict_free_warp_instr_per_sm_clk"]
fp = dict(common, **{k: v for k, v in d.items() if k.startswith(("dadd", "dfma", "f2f", "ffma", "fp64", "dmma"))})
json.dump(smem, open("gpurun_out/peaks_smem.json", "w"), indent=1)
json.dump(fp, open("gpurun_out/peaks_fp64.json", "w"), indent=1)
print(json.dumps(smem)); print(json.dumps(fp))
PY
