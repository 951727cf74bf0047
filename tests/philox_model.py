"""numpy model of the in-kernel random streams (the production RNG contract,
see DESIGN.md and draw_tile in csrc/empc_kernels.cuh): Philox4x32-10 keyed by
the 64-bit seed with counters (0xFFFFFFFF, child, instance, generation) for the
two parent ranks, (gene pair, child, instance, generation) for the 32-bit
crossover / mutation uniforms and (gene pair | 2^31, child, instance,
generation) for the Box-Muller noise pair."""
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

    Per gene pair (2q, 2q+1) of a child: counter (q, child, instance,
    generation) gives the crossover uniforms x / y and the mutation uniforms
    z / w of genes 2q / 2q+1 (Bernoulli: u32 < round(prob 2^32)); counter
    (q | 2^31, ...) gives the Box-Muller cos / sin pair from its z, w."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    child = np.arange(nc)
    x, y, _, _ = philox(0xFFFFFFFF, child, instance, generation, k0, k1)
    parents = np.stack([(x * np.uint64(K)) >> S32, (y * np.uint64(K)) >> S32], axis=1).astype(np.int64)
    g, c = np.meshgrid(np.arange(pm), child, indexing="xy")
    q = (g // 2).astype(np.uint64)
    odd = (g % 2) == 1
    x, y, z, w = philox(q, c, instance, generation, k0, k1)
    thr_c = np.uint64(round(crossover_prob * 2.0**32))
    thr_m = np.uint64(round(mutation_prob * 2.0**32))
    take = np.where(odd, y, x) < thr_c
    mut = np.where(odd, w, z) < thr_m
    _, _, bz, bw = philox(q | np.uint64(0x80000000), c, instance, generation, k0, k1)
    u1 = ((bz >> np.uint64(8)).astype(np.float64) + 1.0) * 2.0**-24
    u2 = (bw >> np.uint64(8)).astype(np.float64) * 2.0**-24
    r = np.sqrt(-2.0 * np.log(u1))
    normal = np.where(odd, r * np.sin(2.0 * np.pi * u2), r * np.cos(2.0 * np.pi * u2))
    return parents, take, mut, normal
