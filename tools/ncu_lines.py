"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, res = None, None, []
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0] and r[0] != "":
        try:
            s = float(r[4] or 0); ie = float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        res.append((s, ie, cur_file, r[0], r[1]))
tot = sum(x[0] for x in res) or 1
print(f"total samples {tot:.0f}")
for s, ie, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% inst={ie:9.0f} {f}:{ln:>5} {src.strip()[:90]}")
