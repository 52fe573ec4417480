"""profiles/traffic.json from the ncu captures of one C2 mixed MGS and one CGSR launch
(one 50-step cycle each; tools/one_solve.py C2 mixed <ortho> 1): DRAM bytes / the byte
model's algorithmic bytes of that launch (bench.model_bytes).  Dev tool:
    python tools/traffic_json.py <mgs.ncu-rep> <cgsr.ncu-rep> <commit>"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import model_bytes  # noqa: E402

N, NNZ = 2097152, 14581760


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    get = lambda k: (float(v[h.index(k)].replace(",", "")), u[h.index(k)])
    return get


def scale(x, unit):
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}[unit]


out = {"source": f"ncu --set full --clock-control none -k regex:solve_kernel -c 1 of tools/one_solve.py C2 mixed "
                 f"<ortho> 1 (one 50-step cycle) on the build of commit {sys.argv[3]}",
       "note": "traffic/algorithmic ratio of that launch; bench.py scales it to each timed launch's algorithmic bytes"}
for ortho, rep in (("mgs", sys.argv[1]), ("cgsr", sys.argv[2])):
    g = raw(rep)
    rd = scale(*g("dram__bytes_read.sum"))
    wr = scale(*g("dram__bytes_write.sum"))
    t = scale(*g("gpu__time_duration.sum"))
    alg = model_bytes(N, NNZ, 4, 0 if ortho == "mgs" else 1, [50])
    out[ortho] = {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes": rd + wr, "algorithmic_bytes": alg,
                  "ratio": (rd + wr) / alg, "kernel_ms": t * 1e3, "algorithmic_GBps": alg / t / 1e9,
                  "dram_GBps": (rd + wr) / t / 1e9}
print(json.dumps(out, indent=1))
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
    f.write("\n")
