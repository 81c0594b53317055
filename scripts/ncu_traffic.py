"""Writes profiles/ncu_expert_traffic.json (the bench line's roofline.traffic)
from an `ncu --set full` capture of ONE fused expert-FFN launch: DRAM bytes
read + written against the launch's algorithmic bytes (U+S)*3*d*f*2, with
the commit and command that produced it (provenance).

usage: python scripts/ncu_traffic.py rep.ncu-rep profile_step.log config K commit "command" [out.json]
(profile_step.log holds the per-layer union sizes of the captured step; the
captured launch is layer 0's, `-s 0 -c 1` on the expert_ffn kernel)."""
import re
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

rep, log, config, K, commit, command = sys.argv[1:7]
out = sys.argv[7] if len(sys.argv) > 7 else "profiles/ncu_expert_traffic.json"
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, r = rows[0], rows[1], rows[2]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def val(name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
kname = r[hdr.index("Kernel Name")].split("(")[0] if "Kernel Name" in hdr else "expert_ffn_kernel"
us = [l for l in open(log) if l.startswith("union sizes")][-1]
U0 = int(re.sub(r"np\.int\d+\((\d+)\)", r"\1", us.split(":", 1)[1]).strip(" []\n").split(",")[0])
shape = cb.preset(config)
alg = (U0 + shape.shared_experts) * 3 * shape.d_model * shape.d_ff * 2
d = {"traffic_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": alg,
     "launch": f"{kname} (fused gate/up + SiLU + down), {config} layer 0, K={K}, U={U0} unique experts",
     "source": os.path.basename(rep), "commit": commit, "command": command,
     "dram_read_bytes": rd, "dram_write_bytes": wr,
     "ratio_traffic_over_algorithmic": (rd + wr) / alg, "ratio_read_over_algorithmic": rd / alg,
     "duration_us": val("gpu__time_duration.sum") if "gpu__time_duration.sum" in hdr else None}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
