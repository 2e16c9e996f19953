"""Per-function SASS opcode histogram of a cubin/.so (cuobjdump -sass)."""
import collections, re, subprocess, sys
so, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); funcs[cur] = collections.Counter(); continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        funcs[cur][m.group(1)] += 1
for f, c in funcs.items():
    if pat in f:
        print(f, sum(c.values()))
        print("  " + ", ".join(f"{k}:{v}" for k, v in c.most_common(40)))
