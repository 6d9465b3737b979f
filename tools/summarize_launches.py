"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
python tools/summarize_launches.py launches.csv [--skip-prefix at::] > profiles/..."""
import collections
import csv
import re
import sys


OURS = ("select_count_kernel", "select_scatter_kernel", "gather_copy_kernel", "f32_to_bf16_kernel", "tc_topk_kernel",
        "threshold_kernel", "threshold_warp_kernel", "threshold_union_kernel", "finalize_warp_kernel", "finalize_cta_kernel", "scan_topk_kernel",
        "merge_kernel", "norms_kernel", "range_threshold_kernel", "range_prefix_kernel", "range_verify_kernel",
        "range_write_kernel", "exact_fallback_kernel", "shadow_kernel", "query16_kernel", "select_finish_kernel")


def short(name):
    """libvrs kernels (namespace vrs::, or their base names when ncu drops the namespace)
    -> 'vrs::<kernel>[<template args>]'; anything else is torch / generation."""
    base = re.sub(r"\(.*", "", name).replace("void ", "").strip()
    mine = "vrs::" in name or any(base.split("<")[0].split("::")[-1] == k for k in OURS)
    if mine and "tc_topk_kernel" in base:
        # template args <ARM, MODE, ROWSCALE, BF, PAIR>: name the mode (+ CTA pairs)
        m = re.search(r"<(\d+), (\d+), (\d+), (\d+)(?:, (\d+))?>", base)
        if m:
            mode = {"0": "main", "1": "probe", "2": "range-count", "3": "range-fill"}[m.group(2)]
            return f"vrs::tc_topk_kernel[{mode}{', pairs' if m.group(5) == '1' else ''}]"
    name = re.sub(r"\(.*", "", name)
    targs = re.search(r"<(.*)>", name)
    name = re.sub(r"<.*", "", name).replace("void ", "")
    name = name.split("::")[-1].strip()
    if mine and targs and ("finalize" in name or "threshold" in name or "exact" in name):   # template variants, e.g. <256, 64>
        name += "<" + targs.group(1) + ">"
    return ("vrs::" + name) if mine else name


def main(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = collections.OrderedDict()
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        ns = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
        seq.append((k, ns, r.get("Grid Size", ""), r.get("Block Size", "")))
    ours = {k: v for k, v in agg.items() if k.startswith("vrs::")}
    tot = sum(v[1] for v in ours.values())
    print(f"# ncu launch list summary ({path}); cold-cache, serialised launches: compare SHARES")
    print("| kernel | launches | total ms | mean us | share of libvrs time |")
    print("|---|---|---|---|---|")
    for k, (n, ns) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {ns / tot:.3f} |")
    other = {k: v for k, v in agg.items() if k not in ours}
    if other:
        print(f"\nother (torch data generation / copies): {sum(v[0] for v in other.values())} launches, "
              f"{sum(v[1] for v in other.values()) / 1e6:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
