"""Aggregate an ncu SASS source CSV by CUDA source line.

usage: python tools/sass_lines.py <ncu-sass.csv> <cubin> <mangled-function> [top]

The SASS csv comes from `ncu -i rep --page source --csv --print-source sass`;
line info comes from `nvdisasm -g -c <cubin>` of the same build (offsets are
relative to the function start).
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, func, mode="both"):
    out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    m, cur, inside, pending = {}, None, False, None
    for ln in out.splitlines():
        if ln.startswith(".text.") or ln.startswith("//----"):
            inside = func in ln
            continue
        if not inside:
            continue
        f = re.search(r'## File "([^"]+)", line (\d+)', ln)
        if f:
            here = f"{f.group(1).split('/')[-1]}:{f.group(2)}"
            c = re.search(r'inlined at "([^"]+)", line (\d+)', ln)
            if c:
                outer = f"{c.group(1).split('/')[-1]}:{c.group(2)}"
                pending = f"{here} <- {outer}" if mode == "both" else (
                    here if mode == "inner" else outer)
                cur = pending
            elif pending is None:
                cur = here
            continue
        a = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            m[int(a.group(1), 16)] = cur
            pending = None
    return m


def line_map_g(cubin, func):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    m, cur, inside = {}, None, False
    for ln in out.splitlines():
        if ln.startswith(".text.") or ln.startswith("//----"):
            inside = func in ln
            continue
        if not inside:
            continue
        f = re.search(r'## File "([^"]+)", line (\d+)', ln)
        if f:
            cur = f"{f.group(1).split('/')[-1]}:{f.group(2)}"
            continue
        a = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    import os
    mode = os.environ.get("MODE", "deep")
    if mode == "deep":  # innermost line (-g) <- outermost call site (-gi)
        inner = line_map_g(sys.argv[2], sys.argv[3])
        outer = line_map(sys.argv[2], sys.argv[3], "outer")
        lm = {a: f"{inner.get(a, '?')} <- {outer.get(a, '?')}" for a in set(inner) | set(outer)}
    else:
        lm = line_map(sys.argv[2], sys.argv[3], mode)
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    base = int(data[0][0], 16)
    inst, stall = collections.Counter(), collections.Counter()

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError):
            return 0.0

    for r in data:
        key = lm.get(int(r[0], 16) - base, "?")
        inst[key] += f(r, "Instructions Executed")
        stall[key] += f(r, "Warp Stall Sampling (All Samples)")
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"{'line':48s} {'inst%':>6s} {'stall%':>6s}")
    for k, _ in sorted(stall.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{k:48s} {100 * inst[k] / ti:6.1f} {100 * stall[k] / ts:6.1f}")


if __name__ == "__main__":
    main()
