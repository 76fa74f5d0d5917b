"""Write profiles/r01_k1_traffic.json from an ncu --set full capture of one K1 launch.
usage: ncu_traffic.py K1.ncu-rep ELEMENTS ALG_BYTES_PER_ELEM_UPDATE [out.json]"""
import csv
import io
import json
import subprocess
import sys

rep, elements, alg = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else "profiles/r01_k1_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, val = rows[0], rows[1], rows[2]


def metric(name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
    return float(val[i].replace(",", "")) * scale


rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
grid = val[hdr.index("launch__grid_size")]
d = {"kernel": "k_rhs_update<3,0> (K1), level-4 launch of macro step 3 (AB3 active), C5 full size",
     "elements": elements, "grid": int(grid), "dram_read_bytes": rd, "dram_write_bytes": wr,
     "bytes_per_launch": rd + wr, "bytes_per_elem_update": round((rd + wr) / elements, 1),
     "algorithmic_bytes_per_elem_update": alg,
     "source": "ncu --set full --clock-control none (%s)" % rep.split("/")[-1]}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
