"""Per-source-line hot spots from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    rows = []
    f = None
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        rows.append((f, int(r[0]), samp, inst, r[1].strip()[:90]))
    ts = sum(x[2] for x in rows) or 1
    ti = sum(x[3] for x in rows) or 1
    print(f"total samples {ts}  total warp-inst {ti}")
    for key, name in ((2, "stall samples"), (3, "instructions")):
        print(f"--- top by {name}")
        for x in sorted(rows, key=lambda x: -x[key])[:top]:
            print(f"{x[0]:>16}:{x[1]:<5} {100*x[2]/ts:5.1f}%s {100*x[3]/ti:5.1f}%i  {x[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def ranges(path, spec):
    """spec: list of (label, file, lo, hi) -> instruction / sample share per range."""
    rows = []
    f = None
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            rows.append((f, int(r[0]), int(r[hdr.index("Warp Stall Sampling (All Samples)")]),
                         int(r[hdr.index("Instructions Executed")])))
        except (ValueError, IndexError):
            continue
    ts = sum(x[2] for x in rows) or 1
    ti = sum(x[3] for x in rows) or 1
    for label, fn, lo, hi in spec:
        s = sum(x[2] for x in rows if x[0] == fn and lo <= x[1] <= hi)
        i = sum(x[3] for x in rows if x[0] == fn and lo <= x[1] <= hi)
        print(f"{label:24s} {100*s/ts:5.1f}% samples {100*i/ti:5.1f}% inst")
