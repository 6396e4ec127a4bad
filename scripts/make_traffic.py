"""Build profiles/roofline_traffic.json from ncu --set full reports: mean DRAM traffic
(dram__bytes_read.sum + dram__bytes_write.sum) per call of a C-ABI entry point - every
kernel captured in one report is one call (e.g. prep + main + finish of the attention
backward) and is summed - averaged over the variants that entry point runs per block.

    python scripts/make_traffic.py evo_gated_attention_bwd gpurun_out/r01_bwd_*.ncu-rep
"""
import json, os, subprocess, sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
entry, reports = sys.argv[1], sys.argv[2:]
vals = []
for r in reports:
    out = subprocess.run([sys.executable, os.path.join(HERE, "scripts", "ncu_extract.py"), r], capture_output=True,
                         text=True).stdout
    ks = [json.loads(line) for line in out.splitlines() if line.strip()]
    vals.append({"report": os.path.basename(r), "kernels": [d["kernel"] for d in ks],
                 "traffic_MB": sum(d["traffic_MB"] for d in ks), "time_us": sum(d["time_us"] for d in ks)})
path = os.path.join(HERE, "profiles", "roofline_traffic.json")
doc = json.load(open(path)) if os.path.exists(path) else {}
doc[entry] = {"traffic_bytes_per_launch": 1e6 * sum(v["traffic_MB"] for v in vals) / len(vals),
              "per_variant": vals,
              "how": "ncu --set full --clock-control none, one launch per variant (scripts/attn_micro.py), "
                     "dram__bytes_read.sum + dram__bytes_write.sum"}
json.dump(doc, open(path, "w"), indent=1)
print(json.dumps(doc[entry], indent=1))
