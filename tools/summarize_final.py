"""Summaries of a closing GPU session (tools/gpu_final.sh) for profiles/:
python tools/summarize_final.py gpurun_out/r02_final profiles r02"""
import csv
import json
import os
import sys

src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]


def jline(path):
    if not os.path.exists(path):
        return None
    for line in open(path):
        if line.startswith("{"):
            try:
                return json.loads(line)
            except Exception:
                pass
    return None


def text(path):
    return open(path).read() if os.path.exists(path) else ""


out = [f"# {tag}: closing GPU session (one B200, `tools/gpu_final.sh`)\n"]
t = text(os.path.join(src, "pytest_gpu.log")).strip().splitlines()
out.append("`pytest -m gpu`: " + (t[-2] if len(t) >= 2 else "?") + "; smoke: " +
           (text(os.path.join(src, "smoke.log")).strip().splitlines() or ["?"])[0] + "\n")
out.append("| config | factor time (s) | GFLOP/s | roofline frac (FP64 DGEMM peak) | e2e GFLOP/s | parity | cpu_baseline |")
out.append("|---|---|---|---|---|---|---|")
for cfg in ("c3", "c2", "c1", "c4", "c5_d3"):
    d = jline(os.path.join(src, f"bench_{cfg}.json"))
    if not d:
        out.append(f"| {cfg} | (no line) | | | | | |")
        continue
    par = d.get("parity") or {}
    e2e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    ft = d.get("factor_time_s", d.get("ms_per_step", 0) / 1e3)
    out.append(f"| {cfg} | {ft:.4f} | {d.get('value') or d.get('value_unchecked') or 0:.1f} | "
               f"{(d.get('roofline') or {}).get('frac', 0):.4f} | {e2e.get('value', 0) or 0:.1f} | "
               f"{par.get('ok', par.get('note', '-'))} (rank mismatches {par.get('rank_mismatches', '-')}) | "
               f"{cb.get('value', 0) or 0:.1f} {cb.get('unit', '')} on {cb.get('cores', '-')} core(s) |")
    json.dump(d, open(os.path.join(dst, f"{tag}_bench_{cfg}.json"), "w"))
r = jline(os.path.join(src, "reference_c3.json"))
if r:
    out.append(f"\nReference arm (`--impl reference`, c3, same config, oracle restatement of hmatdag, "
               f"{(r.get('cpu_baseline') or {}).get('cores', 1)} core): {r.get('factor_time_s', 0):.1f} s per "
               f"factorization, {r.get('value', 0):.1f} GFLOP/s.")
    json.dump(r, open(os.path.join(dst, f"{tag}_reference_c3.json"), "w"))
for f in ("launches.csv", "trace_c2.txt", "trace_c3.txt"):
    if os.path.exists(os.path.join(src, f)):
        open(os.path.join(dst, f"{tag}_{f}"), "w").write(text(os.path.join(src, f)))
open(os.path.join(dst, f"{tag}_final_summary.md"), "w").write("\n".join(out) + "\n")

# ---- DMMA A/B
ab = [f"# {tag}: FP64 tensor-core (DMMA, mma.sync m8n8k4) vs DFMA register tiles for the dense contractions\n",
      "Both arms are the same sources; `-DHMX_DMMA=1` switches every `cta_gemm` (the `@` of "
      "hmatrix.py:126-129, 380, 412, 432 and the compact-WY phases) to `gemm_tiles_dmma` "
      "(`csrc/hmx_device.cuh`).  `tools/ab_gemm.py`: batched products, one CTA per product, 4 per SM.\n",
      "| shape (m x n x k) | DFMA us per CTA-op | DFMA TFLOP/s | DMMA us per CTA-op | DMMA TFLOP/s |", "|---|---|---|---|---|"]
rows = {}
for v in ("_dfma", "_dmma"):
    for line in text(os.path.join(src, f"ab_gemm{v}.log")).splitlines():
        if line.startswith("GEMM"):
            p = line.split()
            rows.setdefault(p[1], {})[v] = (p[4], p[8])
for k, d in rows.items():
    a, b = d.get("_dfma", ("-", "-")), d.get("_dmma", ("-", "-"))
    ab.append(f"| {k} | {a[0]} | {a[1]} | {b[0]} | {b[1]} |")
ab.append("")
for v, name in (("_dfma", "DFMA"), ("_dmma", "DMMA")):
    d = jline(os.path.join(src, f"ab_c2{v}.json"))
    if d:
        par = d.get("parity") or {}
        ab.append(f"c2, one factorization, {name} build: {d.get('factor_time_s', 0):.4f} s, parity ok = {par.get('ok')} "
                  f"(rank mismatches {par.get('rank_mismatches')}).")
ab.append("\nncu counters of one launch of the 256^3 batch (`--metrics`, `k_tasks<1>`):\n")
for v, name in (("_dfma", "DFMA"), ("_dmma", "DMMA")):
    p = os.path.join(src, f"ncu_gemm{v}.csv")
    if not os.path.exists(p):
        continue
    lines = [l for l in open(p) if l.startswith('"')]
    try:
        rd = list(csv.reader(lines))
        hdr = rd[0]
        im, iv, iu = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        ab.append(f"* {name}: " + "; ".join(f"{r_[im]} = {r_[iv]} {r_[iu]}" for r_ in rd[1:]))
    except Exception as e:  # keep the raw file name if the layout differs
        ab.append(f"* {name}: see {p} ({e})")
open(os.path.join(dst, f"{tag}_dmma_ab.md"), "w").write("\n".join(ab) + "\n")
print("\n".join(out))
print("\n".join(ab))
