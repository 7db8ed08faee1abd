"""In-graph launch timeline of the decode step (eeb_debug_stamps).

Every step kernel stamps its first CTA start and last warp exit with
%globaltimer inside the captured, PDL-chained graph (common.cuh StampScope),
so the per-kernel times below come from the same execution as the timed
step, not from a serialised profiler replay.

Attribution: a launch's *critical-path time* is how far it moves the step's
last-finished point, ``crit = max(0, end - max(end of every earlier launch))``.
Kernels overlap under PDL (a GEMM streams weights while its predecessor
drains), so busy spans (end - start) over-count; crit times sum exactly to the
step span (first start -> last end), which is what the roofline fractions in
bench.py are computed from.
"""
from __future__ import annotations

import numpy as np

CATS = ("layer_gemm", "attention", "exit_head", "norm", "other")


def kernel_kind(name: str) -> str:
    for k in ("gemm_tc", "gemm_cc", "attention_dec", "attention_mma", "attention_pipe", "attention_prefill", "attention_kernel",
              "kv_append", "residual_norm", "plane_sum", "act_kernel", "decide", "gather_rows", "finalize",
              "head_reduce", "embed", "mark_depth"):
        if k in name:
            return k
    return name


def analyse(launches: list[dict]) -> dict:
    """Per-launch critical-path times and per-category sums of one step."""
    t0 = min(l["start_ns"] for l in launches if l["ctas"] > 0)
    last = t0
    rows = []
    for l in launches:
        if l["ctas"] <= 0:  # not run (a conditional graph body switched off)
            rows.append({**l, "kind": kernel_kind(l["kernel"]), "crit_ns": 0, "busy_ns": 0, "lat_ns": -1,
                         "work_ns": -1, "tail_ns": -1})
            continue
        crit = max(0, l["end_ns"] - last)
        w = l.get("wait_ns", -1)
        # wait stamped (kernels that record it): launch/flush latency after the
        # predecessor's end, and the work after the wait returned
        lat = w - last if w >= 0 else -1
        work = l["end_ns"] - w if w >= 0 else -1
        mk = l.get("mark_ns", -1)
        tail = l["end_ns"] - mk if mk >= 0 and w >= 0 else -1
        last = max(last, l["end_ns"])
        rows.append({**l, "kind": kernel_kind(l["kernel"]), "crit_ns": crit, "busy_ns": l["end_ns"] - l["start_ns"],
                     "lat_ns": lat, "work_ns": work, "tail_ns": tail})
    span = last - t0
    cats = {}
    for r in rows:
        c = cats.setdefault(r["cat"], {"crit_ns": 0, "busy_ns": 0, "launches": 0})
        c["crit_ns"] += r["crit_ns"]
        c["busy_ns"] += r["busy_ns"]
        c["launches"] += 1
    return {"span_ns": span, "launches": rows, "cats": cats}


def run(ctx, step, n_steps: int, max_launches: int = 1024) -> dict:
    """Stamp `n_steps` calls of step(k) (each one decode step on ctx) and
    average the per-launch times over them (the graph is identical per step)."""
    ctx.stamps(max_launches)
    try:
        per = []
        step(0)  # capture the stamped graph
        ctx.synchronize()
        for k in range(n_steps):
            step(k)
            per.append(analyse(ctx.stamps_read()))
    finally:
        ctx.stamps(0)
    n = len(per[0]["launches"])
    assert all(len(p["launches"]) == n for p in per), "launch list changed between stamped steps"
    crit = np.mean([[r["crit_ns"] for r in p["launches"]] for p in per], axis=0)
    busy = np.mean([[r["busy_ns"] for r in p["launches"]] for p in per], axis=0)
    lat = np.mean([[r["lat_ns"] for r in p["launches"]] for p in per], axis=0)
    work = np.mean([[r["work_ns"] for r in p["launches"]] for p in per], axis=0)
    tail = np.mean([[r["tail_ns"] for r in p["launches"]] for p in per], axis=0)
    ran = np.mean([[1.0 if r["ctas"] > 0 else 0.0 for r in p["launches"]] for p in per], axis=0)
    span = float(np.mean([p["span_ns"] for p in per]))
    launches = [{"kernel": r.get("kind", r["kernel"]), "cat": r["cat"], "ctas": r["ctas"], "ran": float(rn),
                 "crit_us": float(c) / 1e3, "busy_us": float(b) / 1e3,
                 **({"lat_us": float(la) / 1e3, "work_us": float(wo) / 1e3} if r["lat_ns"] >= 0 else {}),
                 **({"tail_us": float(ta) / 1e3} if r["tail_ns"] >= 0 else {})}
                for r, c, b, la, wo, ta, rn in zip(per[0]["launches"], crit, busy, lat, work, tail, ran)]
    cats = {}
    for l in launches:
        c = cats.setdefault(l["cat"], {"crit_ms": 0.0, "busy_ms": 0.0, "launches": 0})
        c["crit_ms"] += l["crit_us"] / 1e3
        c["busy_ms"] += l["busy_us"] / 1e3
        c["launches"] += 1
    return {"steps": n_steps, "span_ms": span / 1e6, "launches": launches, "cats": cats}


def table(tl: dict, top: int = 0) -> str:
    out = [f"step span {tl['span_ms'] * 1e3:.1f} us over {len(tl['launches'])} launches "
           f"(in-graph %globaltimer stamps, mean of {tl['steps']} steps)"]
    for cat, c in sorted(tl["cats"].items(), key=lambda kv: -kv[1]["crit_ms"]):
        out.append(f"  {cat:12s} n={c['launches']:4d}  crit {c['crit_ms'] * 1e3:8.1f} us "
                   f"({100 * c['crit_ms'] / tl['span_ms']:5.1f}%)  busy {c['busy_ms'] * 1e3:8.1f} us")
    if top:
        out.append("  launches (crit / busy us):")
        for i, l in enumerate(tl["launches"][:top]):
            extra = (f"  (wait-after-prev {l['lat_us']:6.2f}, work {l['work_us']:6.2f}" +
                     (f", tail {l['tail_us']:6.2f}" if "tail_us" in l else "") + ")" if "lat_us" in l else "")
            out.append(f"    {i:4d} {l['kernel']:18s} {l['cat']:11s} ctas={l['ctas']:5d} "
                       f"crit {l['crit_us']:7.2f}  busy {l['busy_us']:7.2f}{extra}")
    return "\n".join(out)
