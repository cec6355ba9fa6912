"""Updates profiles/ncu_traffic.json from `ncu --set full` reports of the
bench workload (C5, 256^3 cells): per kernel variant, the DRAM bytes (read +
write) per launch and, for the fused step, its fp64-pipe instructions per
cell.  Each entry carries the hash of the sources that compile into the
kernel (bench.kernel_src_sha16): bench.py reports an entry only while the
sources are unchanged, so a stale number can never reach the bench line.

usage: python tools/traffic_json.py REPORT.ncu-rep [...]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import TRAFFIC_JSON, kernel_src_sha16  # noqa: E402

MAP = {"k_lu_solve": "lu_solve", "k_lu_factor": "lu_setup", "k_adv3d": "advection",
       "k_reduce<1>": "wrms", "k_lincomb<3": "residual", "k_lincomb<4": "rhs_combine",
       "k_cellmap<FJacobian": "jacobian", "k_cellmap_tma<FReaction": "reaction"}
CELLS = 256 ** 3
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def variant_of(name):
    """fused_newton/<numerics> from k_fused_newton<K, KIND, ADV, FIRST, GJ, CT>."""
    m = re.search(r"k_fused_newton<(\d+), (\d+), (\d+), (\d+), (\d+), (\d+)(?:, (\d+))?>", name)
    if not m:
        for key, short in MAP.items():
            if key in name:
                return short + "/composed"
        return None
    gj, ct, tol = int(m.group(5)), int(m.group(6)), int(m.group(7) or 0)
    return "fused_newton/" + ("contracted" if ct else ("exact_gj" if gj else "exact")) + ("_tol" if tol else "")


def fp64_per_cell(rep):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    sh = rows[1]
    iS, iE = sh.index("Source"), sh.index("Instructions Executed")
    n64 = 0
    for r in rows[2:]:
        op = r[iS].split()
        if op:
            o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
            if o in ("DADD", "DMUL", "DFMA", "DSETP"):
                n64 += int(r[iE] or 0)
    return round(n64 * 32 / CELLS, 1)


def main(reports):
    try:
        with open(TRAFFIC_JSON) as f:
            doc = json.load(f)
    except (OSError, ValueError):
        doc = {}
    entries = doc.get("entries", {})
    sha = kernel_src_sha16()
    for rep in reports:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, u = rows[0], rows[1]
        ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        for r in rows[2:]:
            name = r[h.index("Kernel Name")]
            key = variant_of(name)
            if key is None:
                continue
            e = {"dram_bytes": float(r[ir].replace(",", "")) * MULT[u[ir]] +
                 float(r[iw].replace(",", "")) * MULT[u[iw]],
                 "src_sha16": sha, "source": f"ncu --set full --clock-control none, {os.path.basename(rep)}",
                 "kernel_name": name}
            if key.startswith("fused_newton/"):
                e["fp64_per_cell"] = fp64_per_cell(rep)   # the report holds one fused kernel
            entries[key] = e
    doc = {"_doc": __doc__.split("\n\n")[0], "entries": entries}
    with open(TRAFFIC_JSON, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
