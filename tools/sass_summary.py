"""Per-kernel SASS census of librowblock_b200.so (cuobjdump -sass): counts of the Blackwell-native
instructions that prove the tcgen05 / TMA / TMEM paths (UTCHMMA / UTCQMMA = tcgen05.mma, UTMALDG /
UBLKCP = TMA tensor / bulk copies, LDTM / STTM = tcgen05.ld / st, UTCBAR = tcgen05.commit,
SYNCS = mbarrier ops) plus register-file gathers (LDG) and stores (STG), for the kernels of the
hot path.  Usage: python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.txt"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2202_05868_b200/librowblock_b200.so"
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS", "LDGSTS", "LDG", "STG",
       "LDS", "STS", "HMMA"]
HOT = re.compile(r"spmm|sweep|csr|greedy|quotient|vbr|compact|convert|widen|fanout")


def strip_args(d):
    """Drop the trailing parameter list of a demangled name."""
    if not d.endswith(")"):
        return d
    depth = 0
    for i in range(len(d) - 1, -1, -1):
        depth += {")": 1, "(": -1}.get(d[i], 0)
        if depth == 0:
            return d[:i]
    return d


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    rows = []
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if not HOT.search(name):
            continue
        body = f.split("\n", 1)[1] if "\n" in f else ""
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", body)
        cnt = {op: sum(1 for i in ins if i == op) for op in OPS}
        rows.append((name, len(ins), cnt))
    try:
        dem = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
    except FileNotFoundError:
        dem = [r[0] for r in rows]
    print(f"# SASS census of {LIB} (cuobjdump -sass, sm_100a); instruction counts per kernel (static, not executed)")
    print("kernel\tinstrs\t" + "\t".join(OPS))
    for (name, n, cnt), d in zip(rows, dem):
        short = strip_args((d or name).replace("(anonymous namespace)::", ""))
        print(f"{short}\t{n}\t" + "\t".join(str(cnt[o]) for o in OPS))


if __name__ == "__main__":
    main()
