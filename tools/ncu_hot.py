"""Top stalled SASS instructions of each kernel in an .ncu-rep (source page)."""
import csv
import io
import subprocess
import sys


def main(path, top=25):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], text=True)
    blocks = out.split('"Kernel Name"')
    for b in blocks[1:]:
        lines = b.splitlines()
        name = lines[0][:90]
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
        tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
        print("==", name, "samples", tot)
        data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
        for d in data[:top]:
            s = int(d["Warp Stall Sampling (All Samples)"] or 0)
            stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
            top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
            print(f"  {100*s/tot:5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} {top3}")
        break  # first kernel instance only


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
