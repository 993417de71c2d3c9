"""Static SASS footprint of one kernel by source function (nvdisasm -gi line info; innermost frame).

  python tools/sass_static.py <nvdisasm -c -gi output> <mangled kernel> <source.cu> [<header.cuh> ...]
"""
import bisect
import collections
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
    sass, fn, *srcs = sys.argv[1:]
    tabs = {s.split("/")[-1]: functions(s) for s in srcs}
    inside, run, cur = False, [], []
    cnt = collections.Counter()
    for ln in open(sass):
        if ln.startswith("//----") and ".text." in ln:
            inside = f".text.{fn} " in ln or ln.strip().endswith(f".text.{fn}")
            continue
        if not inside:
            continue
        m = re.findall(r'"([^"]+)", line (\d+)', ln) if "//## File" in ln else None
        if m:
            run.append(m)
            continue
        if re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln):
            if run:
                cur = [(f.split("/")[-1], int(l)) for r in run for f, l in r]
                run = []
            f, l = cur[0] if cur else ("?", 0)
            if f in tabs:
                st = tabs[f]
                i = bisect.bisect_right([s[0] for s in st], l) - 1
                cnt[f"{f}:{st[i][1] if i >= 0 else '?'}"] += 1
            else:
                cnt[f] += 1
    tot = sum(cnt.values())
    print("total", tot)
    for k, v in cnt.most_common(30):
        print(f"{v:6d} {k}")


if __name__ == "__main__":
    main()
