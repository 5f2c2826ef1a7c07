"""Per-source-line hot spots of an ncu report (developer tool): warp instructions executed and
warp-stall samples per CUDA source line (the `--page source --print-source cuda,sass` view,
which needs -lineinfo and --import-source on).

    python tools/ncu_lines.py report.ncu-rep [--top 40] [--out summary.txt]
"""
import csv
import io
import subprocess
import sys


def lines(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows = None, None, []
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or not rec[0].isdigit():
            continue  # the SASS rows of a line start with an address
        d = dict(zip(hdr[2:], rec[2:]))
        try:
            inst = int(d.get("Instructions Executed", "0") or 0)
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if inst or samp:
            rows.append((fname, int(rec[0]), rec[1].strip(), inst, samp))
    return rows


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    rows = lines(path)
    ti = sum(r[3] for r in rows) or 1
    ts = sum(r[4] for r in rows) or 1
    buf = [f"{path}: {ti} warp instructions, {ts} stall samples over {len(rows)} source lines",
           f"{'file:line':32s} {'inst%':>6s} {'samp%':>6s}  source"]
    for f, ln, src, inst, samp in sorted(rows, key=lambda r: -r[4])[:top]:
        buf.append(f"{f + ':' + str(ln):32s} {100 * inst / ti:6.2f} {100 * samp / ts:6.2f}  {src[:90]}")
    text = "\n".join(buf)
    print(text)
    if "--out" in sys.argv:
        open(sys.argv[sys.argv.index("--out") + 1], "w").write(text + "\n")


if __name__ == "__main__":
    main()
