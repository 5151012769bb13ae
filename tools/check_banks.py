"""Shared-memory bank-conflict check of decode_attn's fragment reads (design
aid, mirrors the index math of neo_attn.cu: swz(), tok_pi(), the K chunk set
q + 4i and the V chunks r, r + 8).  LDS.128 is served in 4 phases of 8 lanes;
a phase is conflict-free iff its 8 lanes touch 8 distinct 16-byte bank groups.
Run: python tools/check_banks.py  -> prints the worst conflict degree (1 = none)."""


def swz(t, c):
    R = 2 * t + (c >> 3)
    return R * 128 + (((c & 7) ^ (R & 7)) << 4)


def tok_pi(rho):
    return 4 + ((rho >> 1) ^ 2) if rho & 1 else rho >> 1


def worst_degree(addrs):
    worst = 1
    for p in range(4):
        groups = [(addrs[l] % 128) // 16 for l in range(8 * p, 8 * p + 8)]
        worst = max(worst, max(groups.count(g) for g in groups))
    return worst


def k_reads():
    for row in range(2):
        for i in range(4):
            yield [swz(tok_pi(l >> 2) + 8 * row, (l & 3) + 4 * i) for l in range(32)]


def v_reads():
    for e in range(4):
        for f in range(2):
            out = []
            for l in range(32):
                r, q = l >> 2, l & 3
                toks = [tok_pi(2 * q), tok_pi(2 * q + 1), 8 + tok_pi(2 * q), 8 + tok_pi(2 * q + 1)]
                out.append(swz(toks[e], r + 8 * f))
            yield out


def main():
    k = max(worst_degree(a) for a in k_reads())
    v = max(worst_degree(a) for a in v_reads())
    print(f"K worst conflict degree {k}, V worst conflict degree {v}")
    return k, v


if __name__ == "__main__":
    main()
