"""Per-CUDA-source-line totals from an ncu capture (--import-source on, -lineinfo build):
warp-instructions executed and stall samples by file:line, largest first.
python tools/ncu_lines.py capture.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    fname, hdr, out = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[2] == "-":
            try:
                out.append((fname, int(r[0]), r[1].strip(), int(r[7]), int(r[4])))
            except ValueError:
                pass
    ti = sum(o[3] for o in out) or 1
    ts = sum(o[4] for o in out) or 1
    print(f"total warp-instructions {ti / 1e9:.3f} G, stall samples {ts}")
    for f, ln, src, ni, ns in sorted(out, key=lambda o: -o[3])[:top]:
        print(f"{100 * ni / ti:5.2f}% inst {100 * ns / ts:5.2f}% stall  {f}:{ln:<4d} {src[:90]}")


if __name__ == "__main__":
    main()
