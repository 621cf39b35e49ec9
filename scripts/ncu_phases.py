"""Dev tool: summarise an ncu report of tile_filter_kernel by phase
(SASS ranges between barriers) -- stall samples, instructions per pixel,
shared wavefronts vs ideal."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
npx = float(sys.argv[2]) if len(sys.argv) > 2 else 4194304.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
col = {k: hdr.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)", "Instructions Executed",
                                 "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal")}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
rcol = [hdr.index(h) for h in reasons]
stalls = []
data = []
for r in rows[2:]:
    if len(r) <= col["Instructions Executed"]:
        continue
    g = lambda k: int(r[col[k]] or 0) if r[col[k]].strip().isdigit() else 0  # noqa: E731
    data.append((r[col["Source"]], g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"),
                 g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal")))
    stalls.append([int(r[c]) if r[c].strip().isdigit() else 0 for c in rcol])
cuts = [0] + [i + 1 for i, d in enumerate(data) if "BAR.SYNC" in d[0]] + [len(data)]
tot = sum(d[1] for d in data)
print(f"total stall samples {tot}")
for a, b in zip(cuts[:-1], cuts[1:]):
    seg = data[a:b]
    st = sum(d[1] for d in seg)
    if st == 0 and sum(d[2] for d in seg) == 0:
        continue
    ops = collections.Counter()
    for s, _, ex, _, _ in seg:
        t = s.split()
        if not t:
            continue
        o = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[o.split(".")[0]] += ex
    inst = sum(ops.values()) * 32 / npx
    dp = sum(ops[k] for k in ("DADD", "DFMA", "DMUL", "DSETP")) * 32 / npx
    wf = sum(d[3] for d in seg)
    wfi = sum(d[4] for d in seg)
    top = " ".join(f"{k}:{v * 32 / npx:.0f}" for k, v in ops.most_common(8))
    print(f"[{a:5d},{b:5d}) stall {100 * st / max(tot, 1):5.1f}%  inst/px {inst:6.0f}  dp/px {dp:5.0f}  "
          f"smem wf {wf / 1e6:6.2f}M (ideal {wfi / 1e6:6.2f}M)  {top}")
    rs = [sum(x[i] for x in stalls[a:b]) for i in range(len(reasons))]
    rt = sum(rs) or 1
    top_r = sorted(zip(rs, reasons), reverse=True)[:5]
    if st > 0.01 * tot:
        print("        reasons: " + " ".join(f"{n[6:]}:{100 * v / rt:.0f}%" for v, n in top_r if v))
alltot = collections.Counter()
for s_, _, ex, _, _ in data:
    t = s_.split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    alltot[o.split(".")[0]] += ex
tot_inst = sum(alltot.values()) * 32 / npx
tot_dp = sum(alltot[k] for k in ("DADD", "DFMA", "DMUL", "DSETP")) * 32 / npx
print(f"TOTAL inst/px {tot_inst:.0f}  fp64 inst/px {tot_dp:.0f}  smem wavefronts/px "
      f"{sum(d[3] for d in data) / npx:.2f}")
