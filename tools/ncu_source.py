"""Top source lines by warp-stall samples for one kernel of an ncu report."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=15):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    data, tot = [], 0.0
    for r in rows:
        if len(r) > si and r[0] not in ("", "Line No") and r[0].isdigit():
            try:
                v = float(r[si])
            except ValueError:
                continue
            tot += v
            data.append((v, r[0], r[1].strip()[:100]))
    data.sort(reverse=True)
    for v, ln, src in data[:int(top)]:
        print(f"{100 * v / max(tot, 1):5.1f}%  L{ln:>4}  {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
