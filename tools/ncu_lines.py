"""Per-source-line instruction mix and stall samples of an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass), for reading the
fused kernel's hot spots without a GPU."""
import collections
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    per = collections.defaultdict(collections.Counter)
    stall = collections.Counter()
    fname, cur, iE = "?", None, None

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    warps = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            iE = r.index("Instructions Executed")
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1][:60])
            continue
        src = r[3].strip()
        if not src or iE is None:
            continue
        toks = src.split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        per[cur][op] += num(r[iE])
        stall[cur] += num(r[4])
    total = sum(sum(c.values()) for c in per.values())
    print(f"total warp instructions {total}")
    for n, k in sorted(((sum(c.values()), k) for k, c in per.items()), reverse=True)[:top]:
        c = per[k]
        fp = c["DADD"] + c["DMUL"] + c["DFMA"]
        oth = ", ".join(f"{o}:{v / n:.2f}" for o, v in c.most_common(7) if o not in ("DADD", "DMUL", "DFMA"))
        print(f"{k[0][:12]:12s}{k[1]:5d} {100 * n / total:5.1f}% fp64 {100 * fp / max(n, 1):3.0f}% "
              f"stall {stall[k]:6d}  {k[2][:44]:44s} {oth}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
