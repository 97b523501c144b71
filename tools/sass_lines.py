"""Attribute an ncu SASS source page (--page source --csv --print-source sass) to CUDA source lines.

    python tools/sass_lines.py SRC_SASS.csv KERNEL.sass [--top 40]
KERNEL.sass: `nvdisasm -gi` text of the same kernel's .text section (offsets + line info).
Prints instructions executed and stall samples per repo source line (innermost repo frame).
"""
import collections
import csv
import re
import sys


def line_map(path):
    m = {}
    cur = None
    fresh = True          # the first "//## File" line of a group is the innermost frame
    for ln in open(path):
        if ln.lstrip().startswith("//## File"):
            frames = re.findall(r'"([^"]+)", line (\d+)', ln)
            repo = [(f, int(n)) for f, n in frames if "/repo/" in f]
            if repo and fresh:
                cur = (repo[0][0].split("/")[-1], repo[0][1])
                fresh = False
            continue
        fresh = True
        mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if mo:
            m[int(mo.group(1), 16)] = cur
    return m


def main():
    src, sass = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    lm = line_map(sass)
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    sm = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) >= len(hdr) and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    inst = collections.Counter()
    samp = collections.Counter()
    for r in data:
        key = lm.get(int(r[0], 16) - base)
        inst[key] += int(r[ie] or 0)
        samp[key] += int(r[sm] or 0)
    T = sum(inst.values())
    S = sum(samp.values())
    print(f"total {T/1e9:.2f} G warp-inst, {S} samples")
    for key, n in inst.most_common(top):
        print(f"{str(key):28s} inst {n/T*100:5.1f}%  stalls {samp[key]/S*100:5.1f}%")


if __name__ == "__main__":
    main()
