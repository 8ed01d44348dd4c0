"""Write profiles/k5a_traffic_<cfg>.json from an `ncu --set full` capture of K5a:
dram__bytes_read.sum + dram__bytes_write.sum of the captured launch, stamped with the sha of
K5a's sources (bench.py reports the figure only while the sources are unchanged).

    python tools/traffic_from_ncu.py gpurun_out/k5a_cfg4_r02a.ncu-rep cfg4
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def metric(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", name], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    col = hdr.index(name)
    units = rows[1][col]
    vals = [float(r[col].replace(",", "")) for r in rows[2:] if len(r) > col and r[col]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units, 1)
    return [v * scale for v in vals], rows[2][hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"


def main(rep, cfg):
    import bench
    rd, kname = metric(rep, "dram__bytes_read.sum")
    wr, _ = metric(rep, "dram__bytes_write.sum")
    out = {"what": "dram__bytes_read.sum + dram__bytes_write.sum of one K5a launch (%s), ncu --set full" % kname,
           "bytes_per_launch": rd[0] + wr[0], "read": rd[0], "write": wr[0], "source": os.path.basename(rep),
           "k5a_source_sha": bench.k5a_source_sha()}
    path = os.path.join(ROOT, "profiles", "k5a_traffic_%s.json" % cfg)
    json.dump(out, open(path, "w"), indent=1)
    print(path, out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
