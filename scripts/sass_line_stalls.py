"""Attribute an ncu SASS source page (CSV, `--page source --csv`) to CUDA
source lines via `nvdisasm -gi` of the same cubin: per line (innermost
inlined location) the warp-stall samples, top lines printed.

    python scripts/sass_line_stalls.py ncu_sass.csv[.gz] kernel.sass [N] [file-filter]
"""
import csv, gzip, io, re, sys, collections


def main():
    src, sass = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    filt = sys.argv[4] if len(sys.argv) > 4 else ""
    op = gzip.open if src.endswith(".gz") else open
    rows = list(csv.reader(io.TextIOWrapper(op(src, "rb"))))
    h = rows[1]
    ia, isamp = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][ia], 16)
    samples = {int(r[ia], 16) - base: float(r[isamp] or 0) for r in data}
    # offset -> innermost "File, line" annotation
    # an instruction's annotations come innermost first ("... inlined at ...")
    loc, group, cur = {}, [], None
    for line in open(sass):
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            group.append((m.group(1).rsplit("/", 1)[-1], int(m.group(2))))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m:
            if group:
                cur = group[0]
                group = []
            if cur:
                loc[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    tot = sum(samples.values())
    for off, v in samples.items():
        agg[loc.get(off, ("?", 0))] += v
    print(f"total samples {tot:.0f}")
    shown = 0
    for (f, l), v in agg.most_common():
        if filt and filt not in f:
            continue
        print(f"{100 * v / tot:6.2f} %  {f}:{l}")
        shown += 1
        if shown >= top:
            break


if __name__ == "__main__":
    main()
