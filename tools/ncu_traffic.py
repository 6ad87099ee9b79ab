"""Record the DRAM traffic of one kernel launch from an `ncu --set full` report into profiles/traffic.json.

python tools/ncu_traffic.py REPORT KEY SOURCE_NAME
  KEY          config/variant/scatter, e.g. c5/structured/tiled (the key bench.py looks up)
  SOURCE_NAME  the committed summary file the number comes from (profiles/...)
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, src = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))


def val(name):
    v = float(d[name].replace(",", ""))
    u = units.get(name, "")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u, 1.0)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
dur = val("gpu__time_duration.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
try:
    with open(path) as f:
        t = json.load(f)
except Exception:
    t = {}
t[key] = {"kernel": d.get("Kernel Name", "?")[:80], "dram_read_bytes": rd, "dram_write_bytes": wr,
          "dram_bytes": rd + wr, "duration_s_under_ncu": dur, "source": src}
with open(path, "w") as f:
    json.dump(t, f, indent=1, sort_keys=True)
print(json.dumps(t[key]))
