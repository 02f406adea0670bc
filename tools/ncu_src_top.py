"""Top CUDA source lines of one kernel in an ncu report by executed
instructions and stall samples:  python tools/ncu_src_top.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, f, hdr = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] and len(r) > 4 and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        res.append((int(d.get("Instructions Executed", 0) or 0), int(r[4] or 0), f, r[0], r[1][:90]))
tot_i = sum(x[0] for x in res) or 1
tot_s = sum(x[1] for x in res) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for key, name in ((0, "instructions"), (1, "stall samples")):
    print(f"--- by {name}")
    for x in sorted(res, key=lambda x: -x[key])[:n]:
        print(f"{x[0] / tot_i:6.1%} {x[1] / tot_s:6.1%}  {x[2]}:{x[3]}  {x[4]}")
