#!/usr/bin/env python3
"""Per-function SASS opcode histogram of a cubin/.so (cuobjdump -sass)."""
import collections, re, subprocess, sys
lib = sys.argv[1]; pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn, hist = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        fn = m.group(1); hist[fn] = collections.Counter(); continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and fn:
        hist[fn][m.group(2) + (m.group(3) or "")] += 1
for fn, h in hist.items():
    if pat and not pat.search(fn): continue
    tot = sum(h.values())
    print(f"{fn}  total={tot}")
    print("   " + ", ".join(f"{k}:{v}" for k, v in h.most_common(14)))
