"""Plain-text summary of one `ncu --set full` capture (the metrics quoted in
DESIGN.md and profiles/*_ncu.txt): python tools/ncu_text.py REP.ncu-rep"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summarize import METRICS, STALLS  # noqa: E402

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
col = {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}
print("kernel:", col.get("Kernel Name", ("", "?"))[1][:110])
for k in METRICS:
    if k in col:
        print(f"{k:80s} {col[k][0]:>8s} {col[k][1]}")
st = {s: col.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", ("", "nan"))[1]
      for s in STALLS}
print("stall reasons (cycles per issue): " + ", ".join(f"{k} {float(v):.2f}" for k, v in st.items()))
