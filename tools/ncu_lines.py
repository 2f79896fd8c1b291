"""Aggregate an ncu source page (CUDA view) per source line: top lines by
instructions executed and by warp-stall samples."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr, func = [], None, None, ""
for rec in csv.reader(out.splitlines()):
    if not rec: continue
    if rec[0] == "File Path": fname = rec[1].split("/")[-1]; continue
    if rec[0] == "Function Name": func = rec[1]; continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr and rec[0].isdigit() and len(rec) > 3 and rec[2] == "-" and kern in func:
        d = dict(zip(hdr, rec))
        try:
            ins = int(d.get("Instructions Executed", "0") or 0)
            smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if ins or smp: rows.append((fname, int(rec[0]), ins, smp, rec[1].strip()[:90]))
ti = sum(r[2] for r in rows); ts = sum(r[3] for r in rows)
print(f"total warp-instr {ti:.3e}  samples {ts}")
key = 2 if len(sys.argv) > 4 and sys.argv[4] == "ins" else 3
for r in sorted(rows, key=lambda r: -r[key])[:top]:
    print(f"{r[0]:>18}:{r[1]:<4} ins {100*r[2]/ti:5.1f}%  stall {100*r[3]/ts:5.1f}%  {r[4]}")
