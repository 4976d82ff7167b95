"""Per-kernel SASS evidence for the product library: registers, stack,
spills (cuobjdump -res-usage) and counts of the Blackwell instructions the
design rests on (cuobjdump -sass).  Writes a text table; used by
tests/test_capi_cpu.py and committed as profiles/*_sass_summary.txt.

  python tools/sass_summary.py [lib.so] > profiles/r2_sass_summary.txt
"""
import re
import subprocess
import sys

MNEMONICS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR",
             "SYNCS", "WARPSYNC", "BAR", "ATOMG", "REDG", "LDG", "STG", "FFMA", "SHFL"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        return out.stdout.split("\n")[: len(names)]
    except OSError:
        return names


def resources(lib):
    out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True, check=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in line:
            res[name] = {k: int(v) for k, v in re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)}
            name = None
    return res


def sass_counts(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1)
            counts[name] = {k: 0 for k in MNEMONICS}
            continue
        if name is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            op = m.group(1)
            if op in counts[name]:
                counts[name][op] += 1
    return counts


def summary(lib):
    res, cnt = resources(lib), sass_counts(lib)
    names = sorted(set(res) | set(cnt))
    return [(n, d, res.get(n, {}), cnt.get(n, {})) for n, d in zip(names, demangle(names))]


def main():
    if len(sys.argv) > 1:
        lib = sys.argv[1]
    else:
        sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
        import paper_2402_07033_b200 as M
        lib = M.lib_path()
    print(f"# {lib}: per-kernel registers / stack / local and Blackwell instruction counts")
    print("# kernel | REG STACK LOCAL | " + " ".join(MNEMONICS))
    for _, dem, r, c in summary(lib):
        if not c and not r:
            continue
        print(f"{dem} | {r.get('REG', '-')} {r.get('STACK', '-')} {r.get('LOCAL', '-')} | "
              + " ".join(f"{k}={c.get(k, 0)}" for k in MNEMONICS if c.get(k, 0)))


if __name__ == "__main__":
    main()
