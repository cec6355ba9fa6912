"""Writes profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of
each hot kernel, from `ncu --set full` reports of the bench workload (C5,
256^3 cells).  bench.py reports it as roofline.traffic for the dominant
kernel."""
import csv
import io
import json
import subprocess
import sys

MAP = {"k_fused_newton": "fused_newton", "k_lu_solve": "lu_solve", "k_lu_factor": "lu_setup",
       "k_adv3d": "advection", "k_reduce<1>": "wrms", "k_lincomb<3": "residual",
       "k_lincomb<4": "rhs_combine", "k_cellmap<FJacobian": "jacobian",
       "k_cellmap_tma<FReaction": "reaction"}
CELLS = 256 ** 3
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(reports, out):
    res = {}
    for rep in reports:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, u = rows[0], rows[1]
        ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        for r in rows[2:]:
            name = r[h.index("Kernel Name")]
            for key, bench_name in MAP.items():
                if key in name and bench_name not in res:
                    res[bench_name] = (float(r[ir].replace(",", "")) * MULT[u[ir]] +
                                       float(r[iw].replace(",", "")) * MULT[u[iw]])
        # fp64-pipe instructions (DADD, DMUL, DFMA, DSETP) per cell of the
        # fused step, thread level, from the executed-instruction counts of
        # the SASS source page (the report holds one fused kernel)
        if any("k_fused_newton" in r[h.index("Kernel Name")] for r in rows[2:]) and \
                "fused_newton_fp64_per_cell" not in res:
            src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                 capture_output=True, text=True).stdout
            srows = list(csv.reader(io.StringIO(src)))
            sh = srows[1]
            iS, iE = sh.index("Source"), sh.index("Instructions Executed")
            n64 = 0
            for r in srows[2:]:
                op = r[iS].split()
                if op:
                    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
                    if o in ("DADD", "DMUL", "DFMA", "DSETP"):
                        n64 += int(r[iE] or 0)
            res["fused_newton_fp64_per_cell"] = round(n64 * 32 / CELLS, 1)
    res["_source"] = "ncu --set full --clock-control none, bench.py C5 256^3 (" + ", ".join(reports) + ")"
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:], "profiles/ncu_traffic.json")
