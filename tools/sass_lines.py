"""Attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -gi line info.

  python tools/sass_lines.py <ncu_sass.csv> <nvdisasm -c -gi output> <mangled kernel name> [top]
"""
import collections
import csv
import re
import sys


def sass_lines(path, fn):
    out, cur, inside, prev_ann = {}, None, False, False
    for ln in open(path):
        if ln.startswith("//----") and ".text." in ln:
            inside = ln.strip().endswith(f".text.{fn} --------------------------") or f".text.{fn} " in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:  # a run of annotations lists the innermost inlined location first
            if not prev_ann:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
            prev_ann = True
            continue
        prev_ann = False
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    csv_path, sass_path, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lines = sass_lines(sass_path, fn)
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    samp, inst, stall = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall Sampling" in h]
    for d in data:
        key = lines.get(int(d["Address"], 16) - base) or ("?", 0)
        samp[key] += float(d["Warp Stall Sampling (All Samples)"] or 0)
        inst[key] += float(d["Instructions Executed"] or 0)
    ts, ti = sum(samp.values()), sum(inst.values())
    print(f"total samples {ts:.0f}, warp instructions {ti:.3e}")
    for key, v in samp.most_common(top):
        print(f"{v / ts * 100:5.1f}% samples {inst[key] / ti * 100:5.1f}% inst  {key[0]}:{key[1]}")


if __name__ == "__main__":
    main()
