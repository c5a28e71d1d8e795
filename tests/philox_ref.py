"""Independent pure-Python Philox4x32-10 used by the brute-force pins (tests only).

Written from the Random123 description (Salmon et al. SC'11) and pinned by the known-answer
vectors in tests/golden/philox4x32_10_kat.txt; it shares nothing with oracle/ or the library.
"""
M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c[3] ^ k1) & MASK, p0 & MASK]
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return c


def keyed(seed, rr_id, slot):
    return philox4x32_10([rr_id & MASK, rr_id >> 32, slot & MASK, slot >> 32],
                         [seed & MASK, seed >> 32])
