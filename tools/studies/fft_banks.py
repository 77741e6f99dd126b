"""Bank-conflict check of the radix-8/8/4/4 Stockham passes (Q = 1024, 16-byte
complex elements): for every pass, every group of 8 consecutive lanes (one
shared-memory wavefront of 128 B) must touch 8 distinct 16-byte bank slots.
Finds an XOR swizzle per buffer edge (the layout pass p writes and p+1 reads)."""
import itertools

L = 1024


def passes(radices):
    out, ns = [], 1
    for R in radices:
        out.append((R, ns))
        ns *= R
    return out


def loads(R, ns, nthreads):
    acc = []
    for t in range(R):
        acc.append([j + t * (L // R) if j < L // R else None for j in range(nthreads)])
    return acc


def stores(R, ns, nthreads):
    acc = []
    for t in range(R):
        row = []
        for j in range(nthreads):
            if j >= L // R:
                row.append(None)
                continue
            k = j % ns
            row.append((j - k) * R + k + t * ns)
        acc.append(row)
    return acc


def conflicts(access_rows, sw):
    bad = 0
    for row in access_rows:
        for g in range(0, len(row), 8):
            slots = [sw(a) % 8 for a in row[g:g + 8] if a is not None]
            bad += len(slots) - len(set(slots))
    return bad


def swz(shift, mask=7):
    return lambda i: i ^ ((i >> shift) & mask)


cands = {f"xor>>{s}": swz(s) for s in range(2, 9)}
cands["none"] = lambda i: i
cands["xor>>2^>>5"] = lambda i: i ^ ((i >> 2) & 7) ^ ((i >> 5) & 7)
cands["xor>>3^>>6"] = lambda i: i ^ ((i >> 3) & 7) ^ ((i >> 6) & 7)
cands["xor>>2^>>6"] = lambda i: i ^ ((i >> 2) & 7) ^ ((i >> 6) & 7)

for name, rad in (("inverse", [8, 8, 4, 4]), ("forward", [4, 4, 8, 8])):
    ps = passes(rad)
    print(name, ps)
    for p in range(len(ps) - 1):
        R, ns = ps[p]
        R2, ns2 = ps[p + 1]
        nt_w = 256 if R == 4 else 128
        nt_r = 256 if R2 == 4 else 128
        st = stores(R, ns, nt_w)
        ld = loads(R2, ns2, nt_r)
        ok = [n for n, f in cands.items() if conflicts(st, f) == 0 and conflicts(ld, f) == 0]
        print(f"  edge {p}->{p+1} (R{R} ns{ns} -> R{R2} ns{ns2}): conflict-free swizzles {ok}")

# synthesis input stores / analysis output gathers: lane t owns modes k = t + 1 + 256 i,
# touching positions k and Q - k
sw = cands["xor>>2^>>5"]
rows = []
for i in range(2):
    rows.append([t + 1 + 256 * i if t + 1 + 256 * i < L else None for t in range(256)])
    rows.append([L - (t + 1 + 256 * i) if t + 1 + 256 * i <= L // 2 else None for t in range(256)])
print("mode-owner accesses, xor>>2^>>5: conflicts", conflicts(rows, sw), "| xor>>2:", conflicts(rows, cands["xor>>2"]))
