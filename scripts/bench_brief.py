"""One-line summaries of the bench JSON lines in a gpurun_out directory."""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "bench*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "unparsable", e)
        continue
    r = d.get("roofline", {})
    print(os.path.basename(f), d.get("config", {}).get("kernel_variant"), "value %.1f TF" % (d["value"] / 1e3),
          "kernel_ms %.2f" % r.get("kernel_ms", 0), "frac %.3f" % r.get("frac", 0), "clk", d.get("clocks", {}).get("sm_mhz"))
