"""Top stalled SASS lines of one kernel in an ncu report (reads `--page source --csv`)."""
import csv
import subprocess
import sys


def main(rep, kernel, top=25):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()[1:]))
    h = rows[0]
    ix = h.index("Warp Stall Sampling (All Samples)")
    stalls = [i for i, x in enumerate(h) if x.startswith("stall_")]
    body = [x for x in rows[1:] if len(x) == len(h) and x[ix].replace(".", "").isdigit()]
    total = sum(float(x[ix] or 0) for x in body)
    body.sort(key=lambda x: -float(x[ix] or 0))
    for x in body[:top]:
        why = sorted(((float(x[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:2]
        print(f"{100 * float(x[ix]) / total:5.1f}%  {x[1].strip()[:70]:70s} "
              + " ".join(f"{n}={v:.0f}" for v, n in why if v))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
