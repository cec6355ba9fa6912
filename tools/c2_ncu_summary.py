"""C2 evidence: ncu DRAM bytes per N_Vector op launch at
n = 1e8 .. 1e9 against the algorithmic bytes.  Inputs: the ncu --csv launch
log of `tools/sweep_c2.py --min 1e8 --reps 1 --no-oracle` (6 launches of
the op kernel per sweep row: 5 warm-up + 1 timed) and the sweep's JSON
lines.  ncu times are serialised, cold-cache launches: for the ratio, not
for throughput claims.
Usage: python tools/c2_ncu_summary.py launches.csv sweep.jsonl"""
import csv
import json
import statistics
import sys

BPE = {"N_VLinearSum": 24, "N_VScale": 16, "N_VProd": 24, "N_VDiv": 24, "N_VWrmsNorm": 16,
       "N_VDotProd": 16, "N_VLinearCombination8": 72, "N_VDotProdMulti8": 72,
       "N_VScaleAddMulti8": 136}
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "nsecond": 1e-9, "msecond": 1e-3}


def main(csv_path, jsonl_path):
    rows = [r for r in csv.reader(open(csv_path)) if r and not r[0].startswith("==")]
    h = rows[0]
    iid, ik, im, iu, iv = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                                 "Metric Value"))
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[iid]), {"kernel": r[ik]})
        d[r[im]] = float(r[iv].replace(",", "")) * MULT.get(r[iu], 1.0)
    seq = [launches[k] for k in sorted(launches)]
    sweep = [json.loads(line) for line in open(jsonl_path) if line.strip()]
    print(f"{'op':24s} {'n':>11s} {'kernel':28s} {'alg MB':>9s} {'DRAM MB':>9s} {'DRAM/alg':>8s} "
          f"{'ncu us':>8s} {'ncu GB/s':>9s}")
    for i, row in enumerate(sweep):
        grp = seq[6 * i:6 * i + 6]
        if len(grp) < 6:
            break
        alg = BPE[row["op"]] * row["n"]
        dram = statistics.median(g["dram__bytes_read.sum"] + g["dram__bytes_write.sum"] for g in grp)
        t = statistics.median(g["gpu__time_duration.sum"] for g in grp)
        name = grp[-1]["kernel"].split("(")[0].replace("void ", "")[:28]
        print(f"{row['op']:24s} {row['n']:11d} {name:28s} {alg / 1e6:9.1f} {dram / 1e6:9.1f} "
              f"{dram / alg:8.3f} {t * 1e6:8.1f} {alg / t / 1e9:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
