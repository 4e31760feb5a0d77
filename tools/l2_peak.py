"""profiles/l2_peak.json from tools/l2bw.cu's output (the best L2-resident size).
usage: python tools/l2_peak.py gpurun_out/l2bw.log"""
import json
import os
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
best = max((r for r in rows if r["bytes"] <= (64 << 20)), key=lambda r: r["gbs"])
out = {"gbs": round(best["gbs"], 1), "bytes": best["bytes"], "all": rows,
       "source": "measured: tools/l2bw.cu (148 x 1024 persistent grid, int4 __ldcg loads, 4 in flight "
                 "per thread, buffer L2-resident after a warm pass; best of 5)"}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                 "l2_peak.json"), "w"), indent=1)
print(out["gbs"], "GB/s")
