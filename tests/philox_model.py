"""numpy model of the in-kernel random streams (the production RNG contract,
see DESIGN.md): Philox4x32-10 keyed by the 64-bit seed with counters
(gene pair, child, instance, generation) for crossover / mutation / noise and
(0xFFFFFFFF, child, instance, generation) for the two parent ranks."""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox(c0, c1, c2, c3, k0, k1):
    c = [np.asarray(x, np.uint64) & MASK for x in (c0, c1, c2, c3)]
    shape = np.broadcast(*c).shape
    c = [np.broadcast_to(x, shape).copy() for x in c]
    k0, k1 = np.uint64(k0) & MASK, np.uint64(k1) & MASK
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [((p1 >> S32) ^ c[1] ^ k0) & MASK, p1 & MASK, ((p0 >> S32) ^ c[3] ^ k1) & MASK, p0 & MASK]
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return c


def breed_draws(seed, generation, nc, pm, K, crossover_prob, mutation_prob, instance=0):
    """parents (nc, 2) ranks, take (nc, pm), mutate (nc, pm), z (nc, pm) standard normals.

    One Philox call per gene pair (2q, 2q+1) with counter (q, child, instance,
    generation): 16-bit crossover / mutation uniforms from x / y (low half
    for gene 2q, high half for 2q+1), Box-Muller cos / sin pair from z, w."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    child = np.arange(nc)
    x, y, _, _ = philox(0xFFFFFFFF, child, instance, generation, k0, k1)
    parents = np.stack([(x * np.uint64(K)) >> S32, (y * np.uint64(K)) >> S32], axis=1).astype(np.int64)
    g, c = np.meshgrid(np.arange(pm), child, indexing="xy")
    x, y, z, w = philox(g // 2, c, instance, generation, k0, k1)
    shift = (np.uint64(16) * (g % 2).astype(np.uint64))
    thr_c = np.uint64(round(crossover_prob * 2.0**16))
    thr_m = np.uint64(round(mutation_prob * 2.0**16))
    take = ((x >> shift) & np.uint64(0xFFFF)) < thr_c
    mut = ((y >> shift) & np.uint64(0xFFFF)) < thr_m
    u1 = ((z >> np.uint64(8)).astype(np.float64) + 1.0) * 2.0**-24
    u2 = (w >> np.uint64(8)).astype(np.float64) * 2.0**-24
    r = np.sqrt(-2.0 * np.log(u1))
    normal = np.where(g % 2 == 0, r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2))
    return parents, take, mut, normal
