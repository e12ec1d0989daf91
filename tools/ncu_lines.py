"""Per-source-line warp-stall breakdown of an ncu report (needs -lineinfo and --import-source on).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, acc = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            try:
                s = int(r[4])
            except ValueError:
                continue
            st = {}
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h:
                    try:
                        v = int(r[i])
                    except ValueError:
                        continue
                    if v:
                        st[h[6:]] = v
            acc.append((s, cur, int(r[0]), r[1].strip()[:80], st, r[7]))
    tot = sum(a[0] for a in acc) or 1
    acc.sort(key=lambda a: -a[0])
    print(f"total samples {tot}")
    for s, f, ln, src, st, ninst in acc[:top]:
        reasons = ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
        print(f"{100 * s / tot:5.1f}% {f}:{ln} inst={ninst} [{reasons}] {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
