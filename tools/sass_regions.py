"""Attribute ncu SASS samples/instructions to code regions: the innermost raster_fwd.cu / raster_bwd.cu line of each
instruction's inline chain, bucketed by the enclosing function (line ranges from the source).

  python tools/sass_regions.py <ncu_sass.csv> <nvdisasm -c -gi output> <mangled kernel> <source.cu>
"""
import bisect
import collections
import csv
import re
import sys


def functions(src):
    starts = []
    for i, ln in enumerate(open(src), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__|static|__host__)[^(]*?\b(\w+)\(", ln)
        if m:
            starts.append((i, m.group(1)))
    return starts


def main():
    csv_path, sass_path, fn, src = sys.argv[1:5]
    srcname = src.split("/")[-1]
    starts = functions(src)
    lines = [s[0] for s in starts]
    chains, run, inside = {}, [], False
    for ln in open(sass_path):
        if ln.startswith("//----") and ".text." in ln:
            inside = f".text.{fn} " in ln or ln.strip().endswith(f".text.{fn}")
            continue
        if not inside:
            continue
        m = re.findall(r'"([^"]+)", line (\d+)', ln) if "//## File" in ln else None
        if m:
            run.append(m)
            continue
        mm = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if mm:
            if run:
                chain = [(f.split("/")[-1], int(l)) for r in run for f, l in r]
                chains["cur"] = chain
            run = []
            chains[int(mm.group(1), 16)] = chains.get("cur", [])
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    samp, inst = collections.Counter(), collections.Counter()
    fp64 = collections.Counter()  # per (region, opcode): fp64-pipe instructions (D* ops, conversions to/from F64)
    for d in data:
        chain = chains.get(int(d["Address"], 16) - base, [])
        own = [l for f, l in chain if f == srcname]
        if own:
            i = bisect.bisect_right(lines, own[0]) - 1
            region = starts[i][1] if i >= 0 else "?"
        else:
            region = "?"
        samp[region] += float(d["Warp Stall Sampling (All Samples)"] or 0)
        inst[region] += float(d["Instructions Executed"] or 0)
        op = d["Source"].split()[0] if d["Source"].split() else ""
        if op.startswith("@"):
            op = d["Source"].split()[1]
        if re.match(r"D(ADD|MUL|FMA|SETP|MNMX|MMA)", op) or ("F64" in op and op.split(".")[0] in ("F2F", "I2F", "F2I")):
            fp64[(region, op.split(".")[0])] += float(d["Instructions Executed"] or 0)
    ts, ti = sum(samp.values()), sum(inst.values())
    for k, v in samp.most_common():
        print(f"{v / ts * 100:5.1f}% samples {inst[k] / ti * 100:5.1f}% inst  {k}")
    tf = sum(fp64.values())
    if tf:
        print(f"fp64-pipe instructions: {tf:.3e} ({tf / ti * 100:.1f}% of all)")
        for (region, op), v in fp64.most_common(25):
            print(f"  {v / tf * 100:5.1f}%  {region:24s} {op}")


if __name__ == "__main__":
    main()
