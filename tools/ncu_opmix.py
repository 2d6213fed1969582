"""Executed-instruction mix (by SASS opcode) and the top stall sites of a
one-kernel ncu report captured with --import-source on (source page)."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
iS, iE, iN = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
stall = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
mix, samp, tot, sites = collections.Counter(), collections.Counter(), 0, []
for r in rows[h + 1:]:
    try:
        e, n = int(r[iE]), int(r[iN])
    except (ValueError, IndexError):
        continue
    src = r[iS]
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    mix[op] += e
    samp[op] += n
    tot += e
    top = sorted(((hdr[i], int(r[i])) for i in stall if r[i] not in ("", "0")), key=lambda x: -x[1])[:1]
    sites.append((n, src[:60], top))
print("  instruction mix:", ", ".join(f"{o} {100 * c / max(tot, 1):.1f}%" for o, c in mix.most_common(10)))
ns = sum(samp.values()) or 1
print("  warp samples by opcode:", ", ".join(f"{o} {100 * c / ns:.0f}%" for o, c in samp.most_common(6)))
for n, src, top in sorted(sites, key=lambda x: -x[0])[:5]:
    print(f"    {100 * n / ns:4.1f}% {src}  {top}")
