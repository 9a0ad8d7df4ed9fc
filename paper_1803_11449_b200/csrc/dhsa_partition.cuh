// dhsa_partition.cuh -- K1, scan mode 5: the scan behind per-SM shared-memory key tables.
//
// Why.  ncu pins both earlier scan kernels on scattered L2 sectors: k_scan_vec4 needs R
// per packet, k_scan_flowcache one (its pair table lives in L2), and the chip serves
// ~288 G random sectors/s however the SMs ask.  A repeated packet can only be dropped
// for less than one L2 sector if the "seen before" table sits in shared memory -- and a
// window's keys only fit the 148 x 128 KiB of tables if every SM owns a slice of the key
// space.  So this kernel routes each packet to the SM that owns its key, through L2, in
// coalesced runs, and dedups there:
//
//   key        a packet's R bits depend on (cand, h1(opp)) only (_core.pyx:78-86), so the
//              dedup key is the pair (cand, h = h1(opp)): 42 bits at the defaults, not 64,
//              and a scanner's thousands of flows collapse to at most g keys.
//   bijection  A = fmix32(cand ^ h * C) (an invertible 32-bit finaliser), B = h ^ bits of A.
//              bucket b = floor(A * NB / 2^32) is the owning CTA; what is left,
//              rem = (A - lo(b)) << log2(g) | B, still determines (cand, h).  rem's low 13
//              bits pick a 4-way set of 32-bit entries, the rest is the tag, so
//              (bucket, set, tag) identifies the key exactly: a table hit is never a
//              different key, and a missed key is rebuilt from rem by the inverse.
//   producers  PW warps per CTA read tiles of 3584 packets (16-byte loads), bin them by
//              bucket in shared memory (one shared atomic per packet) and copy each bin as
//              one 256-byte slot -- word 0 the count, then up to 31 rems -- into a ring of
//              three chunk buffers in global memory (L2-resident: it is rewritten before it
//              is evicted).  Slots are addressed by (chunk, tile, bucket): no global
//              atomics, aligned 16-byte stores.  A packet whose bin is full goes to a small
//              overflow list that the producers update directly, densely, after the tile.
//   consumers  CW warps per CTA read the slots of their own bucket, four slots per trip,
//              one 8-byte entry per lane, probe the table -- first-choice set, then a second
//              set derived from the tag -- and drop the packet on a hit.  Misses are queued
//              per warp and drained 32 at a time, one per lane: record the key in an empty
//              way of either set, rebuild (cand, h), test + warp-aggregated RED as in the
//              other kernels.
//   flow       producers run up to two chunks ahead of the slowest consumer; the two roles
//              meet only through per-chunk arrival counters (release/acquire), never a
//              grid-wide barrier.
//
// Exactness does not depend on what the tables hold: an entry is written only by a lane
// that issues the key's own update right after, the tables die with the launch, and a
// key that finds both sets full, a bin that overflows or an entry lost to a racing insert
// all end in the direct test + RED.  The result is the same bit array as
// Backend.update_batch (pkg/src/dhsa/_core.pyx:75-86) for any input.
#pragma once
#include "dhsa_device.cuh"

namespace dhsa {

#define DHSA_PT_SETS 8192u          // 4-way sets of u32 entries: 128 KiB of shared memory
#define DHSA_PT_LOG2_SETS 13
#define DHSA_PT_SLOT_WORDS 32u      // one slot = 256 B: word 0 = count, words 1..31 = entries
#define DHSA_PT_SLOT_CAP 31u
#define DHSA_PT_MAX_BUCKETS 160u
#ifndef DHSA_PT_PWARPS
#define DHSA_PT_PWARPS 14           // producer warps per CTA
#endif
#define DHSA_PT_CWARPS (32 - DHSA_PT_PWARPS)  // consumer warps per CTA
#define DHSA_PT_VECS 2              // 16-byte vectors (4 packets each) per producer thread per tile
#define DHSA_PT_TILE_VEC (DHSA_PT_PWARPS * 32 * DHSA_PT_VECS)
#define DHSA_PT_RING 3              // chunk buffers
#define DHSA_PT_TRIP 4              // slots per consumer warp trip
#define DHSA_PT_QUEUE (32 + 32 * DHSA_PT_TRIP)  // queued misses per consumer warp
#define DHSA_PT_OVF 1024u           // overflow list of a tile (packets whose bin was full)

#define DHSA_PT_SMEM_TABLE (DHSA_PT_SETS * 16u)
#define DHSA_PT_SMEM_REGION (DHSA_PT_MAX_BUCKETS * DHSA_PT_SLOT_WORDS * 8u)
#define DHSA_PT_SMEM_QUEUE (DHSA_PT_CWARPS * DHSA_PT_QUEUE * 8u)
#define DHSA_PT_SMEM_OVF (DHSA_PT_OVF * 8u)
#define DHSA_PT_SMEM_LO ((DHSA_PT_MAX_BUCKETS + 4u) * 4u)
#define DHSA_PT_SMEM_CNT ((DHSA_PT_MAX_BUCKETS + 4u) * 4u)
#define DHSA_PT_SMEM_BYTES                                                                              \
    (DHSA_PT_SMEM_TABLE + DHSA_PT_SMEM_REGION + DHSA_PT_SMEM_QUEUE + DHSA_PT_SMEM_OVF + DHSA_PT_SMEM_LO + \
     DHSA_PT_SMEM_CNT)

struct PartParams {
    unsigned long long *ring;   // DHSA_PT_RING x (tiles_per_cta * nb * nb) slots of 32 words
    unsigned int *sync;         // [0..3] chunks produced, [4..7] chunks consumed (arrival counters)
    unsigned long long *stats;  // [0] keys looked up, [1] table hits, [2] packets updated by a producer, [3] keys not recorded
    uint32_t tiles_per_cta;     // tiles every CTA produces per chunk
};

__device__ __forceinline__ void bar_sync_named(int id, int count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_inc(unsigned int *p)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

__device__ __forceinline__ void pt_wait_ge(const unsigned int *p, unsigned int target)
{
    while (ld_acquire_u32(p) < target) __nanosleep(40);
}

// slots are rewritten every DHSA_PT_RING chunks by other SMs: never through L1
__device__ __forceinline__ unsigned long long ld_slot_word(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// the direct update of one key: test each of its R words, RED where the bit is clear
template <int R>
__device__ __forceinline__ void pt_update_direct(uint32_t *__restrict__ words, const DevParams &p, int wshift,
                                                 uint32_t cand, uint32_t h)
{
    const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ (uint64_t)cand) & p.kmask;
    const uint32_t mask = 1u << (h & 31u);
    uint32_t widx[R], w[R];
    packet_slots<R>(p, wshift, cand, h, d0, widx);
#pragma unroll
    for (int i = 0; i < R; i++) w[i] = ld_sketch(words + widx[i]);
#pragma unroll
    for (int i = 0; i < R; i++)
        if ((w[i] & mask) == 0) red_or(words + widx[i], mask);
}

// Drain up to 32 queued keys, one per lane (called by a whole warp): look the key up again
// (another lane may have recorded it since), record it in an empty way of either set, then
// rebuild (cand, h) and update the sketch.
template <int R>
__device__ __forceinline__ void pt_drain32(uint32_t *__restrict__ words, const DevParams &p, int wshift,
                                           uint32_t lo32, uint4 *table, const unsigned long long *q,
                                           uint32_t n_active, uint32_t lane, uint32_t &unstored)
{
    bool act = lane < n_active;
    const unsigned long long rem = act ? q[lane] : 0ull;
    const uint32_t set1 = (uint32_t)rem & (DHSA_PT_SETS - 1u);
    const uint32_t tag = (uint32_t)(rem >> DHSA_PT_LOG2_SETS);
    const uint32_t e1 = (tag << 1) + 1u, e2 = e1 + 1u;
    const uint32_t set2 = set1 ^ ((tag * 0x9E3779B1u) >> (32 - DHSA_PT_LOG2_SETS));
    if (act) {
        const uint4 s1 = table[set1], s2 = table[set2];
        const bool present = s1.x == e1 || s1.y == e1 || s1.z == e1 || s1.w == e1 || s2.x == e2 || s2.y == e2 ||
                             s2.z == e2 || s2.w == e2;
        if (present) {
            act = false;  // recorded by a lane that also issues the update
        } else {
            uint32_t slot_idx = 0xFFFFFFFFu, ent = e2;
            if (s2.w == 0u) slot_idx = set2 * 4u + 3u;
            if (s2.z == 0u) slot_idx = set2 * 4u + 2u;
            if (s2.y == 0u) slot_idx = set2 * 4u + 1u;
            if (s2.x == 0u) slot_idx = set2 * 4u + 0u;
            if (s1.w == 0u) slot_idx = set1 * 4u + 3u, ent = e1;
            if (s1.z == 0u) slot_idx = set1 * 4u + 2u, ent = e1;
            if (s1.y == 0u) slot_idx = set1 * 4u + 1u, ent = e1;
            if (s1.x == 0u) slot_idx = set1 * 4u + 0u, ent = e1;
            if (slot_idx != 0xFFFFFFFFu) reinterpret_cast<uint32_t *>(table)[slot_idx] = ent;
            else unstored++;
        }
    }
    // invert the bijection
    const uint32_t a = (uint32_t)(rem >> p.log2g) + lo32;
    const uint32_t h = ((uint32_t)rem ^ (a >> 11)) & p.gmask;
    const uint32_t cand = unfmix32(a) ^ (h * DHSA_KEY_MUL);
    const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ (uint64_t)cand) & p.kmask;
    const uint32_t mask = 1u << (h & 31u);
    uint32_t widx[R], w[R];
    packet_slots<R>(p, wshift, cand, h, d0, widx);
#pragma unroll
    for (int i = 0; i < R; i++) w[i] = act ? ld_sketch(words + widx[i]) : 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < R; i++) red_or_aggregated(words, widx[i], mask, (w[i] & mask) == 0, lane);
}

template <int R, typename SRC>
__global__ void __launch_bounds__((DHSA_PT_PWARPS + DHSA_PT_CWARPS) * 32, 1)
    k_scan_partition(SRC src, uint32_t *__restrict__ words, DevParams p, PartParams pp)
{
    extern __shared__ __align__(16) uint8_t pt_smem[];
    uint4 *table = reinterpret_cast<uint4 *>(pt_smem);
    unsigned long long *region = reinterpret_cast<unsigned long long *>(pt_smem + DHSA_PT_SMEM_TABLE);
    unsigned long long *queue_s = region + DHSA_PT_MAX_BUCKETS * DHSA_PT_SLOT_WORDS;
    unsigned long long *ovf_s = queue_s + DHSA_PT_CWARPS * DHSA_PT_QUEUE;
    uint32_t *lo_s = reinterpret_cast<uint32_t *>(ovf_s + DHSA_PT_OVF);
    uint32_t *cnt_s = lo_s + DHSA_PT_MAX_BUCKETS + 4u;  // [nb] = overflow list length

    const uint32_t nb = gridDim.x, x = blockIdx.x;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const int wshift = p.log2g - 5;

    for (uint32_t i = tid; i < DHSA_PT_SETS; i += blockDim.x) table[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t i = tid; i < nb; i += blockDim.x)  // lo(b) = ceil(b * 2^32 / nb)
        lo_s[i] = (uint32_t)((((unsigned long long)i << 32) + nb - 1) / nb);
    for (uint32_t i = tid; i <= nb; i += blockDim.x) cnt_s[i] = 0u;
    __syncthreads();

    const uint64_t nvec = src.vectors();
    const uint64_t ntiles = (nvec + DHSA_PT_TILE_VEC - 1) / DHSA_PT_TILE_VEC;
    const uint32_t tpc = pp.tiles_per_cta;
    const uint64_t tiles_per_chunk = (uint64_t)nb * tpc;
    const uint64_t nchunks = (ntiles + tiles_per_chunk - 1) / tiles_per_chunk;
    const uint64_t slots_per_chunk = tiles_per_chunk * nb;

    if (warp < DHSA_PT_PWARPS) {
        // ------------------------------------------------------------ producers --
        constexpr int NPT = DHSA_PT_PWARPS * 32;
        const uint64_t pol = policy_evict_first();
        const H1Consts hc = h1_consts(p.state_h1);
        uint32_t on_time = 0, late = 0;
        unsigned long long direct = 0;
        typename SRC::Raw raw[DHSA_PT_VECS];
#pragma unroll
        for (int v = 0; v < DHSA_PT_VECS; v++)  // tile of (chunk 0, j 0)
            src.load(raw[v], (uint64_t)x * DHSA_PT_TILE_VEC + (uint64_t)v * NPT + tid, pol);
        for (uint64_t c = 0; c < nchunks; c++) {
            if (c >= DHSA_PT_RING && tid == 0)  // the buffer's previous chunk must be consumed everywhere
                pt_wait_ge(pp.sync + 4 + ((c - DHSA_PT_RING) & 3u), nb * (unsigned int)((c - DHSA_PT_RING) / 4 + 1));
            unsigned long long *ring_c = pp.ring + (c % DHSA_PT_RING) * slots_per_chunk * DHSA_PT_SLOT_WORDS;
            for (uint32_t j = 0; j < tpc; j++) {
                const uint64_t tt = (uint64_t)j * nb + x;
                const uint64_t g = c * tiles_per_chunk + tt;
                typename SRC::Raw cur[DHSA_PT_VECS];
#pragma unroll
                for (int v = 0; v < DHSA_PT_VECS; v++) cur[v] = raw[v];
                {  // prefetch this CTA's next tile
                    const uint64_t gn = (j + 1 < tpc) ? g + nb : (c + 1) * tiles_per_chunk + x;
#pragma unroll
                    for (int v = 0; v < DHSA_PT_VECS; v++)
                        src.load(raw[v], gn * DHSA_PT_TILE_VEC + (uint64_t)v * NPT + tid, pol);
                }
                bar_sync_named(1, NPT);  // bins are free again (and the ring buffer, at a chunk's first tile)
                if (g >= ntiles) continue;  // uniform over the CTA
#pragma unroll
                for (int v = 0; v < DHSA_PT_VECS; v++) {
                    uint32_t cs[4], os[4];
                    bool ok[4];
                    src.unpack(cur[v], g * DHSA_PT_TILE_VEC + (uint64_t)v * NPT + tid, cs, os, ok, on_time, late);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t h = h1_fast(hc, os[q], p.gmask);
                        const uint32_t a = fmix32(cs[q] ^ (h * DHSA_KEY_MUL));
                        const uint32_t b = __umulhi(a, nb);
                        const uint32_t bl = (h ^ (a >> 11)) & p.gmask;
                        const unsigned long long rem = ((unsigned long long)(a - lo_s[b]) << p.log2g) | bl;
                        if (ok[q]) {
                            const uint32_t pos = atomicAdd(cnt_s + b, 1u);
                            if (pos < DHSA_PT_SLOT_CAP) {
                                region[b * DHSA_PT_SLOT_WORDS + 1u + pos] = rem;
                            } else {  // the bin is full: the packet goes to the tile's overflow list
                                const uint32_t op = atomicAdd(cnt_s + nb, 1u);
                                if (op < DHSA_PT_OVF) ovf_s[op] = ((unsigned long long)cs[q] << 32) | h;
                                else pt_update_direct<R>(words, p, wshift, cs[q], h), direct++;
                            }
                        }
                    }
                }
                bar_sync_named(1, NPT);
                {
                    // copy the bins out, one 256-byte slot per half-warp trip: a lane moves words 2s, 2s+1
                    unsigned long long *tile_slots = ring_c + tt * nb * DHSA_PT_SLOT_WORDS;
                    const uint32_t half = lane >> 4, sub = lane & 15u;
                    for (uint32_t b0 = 2u * warp; b0 < nb; b0 += 2u * DHSA_PT_PWARPS) {
                        const uint32_t b = b0 + half;
                        uint32_t n = 0;
                        ulonglong2 w2 = make_ulonglong2(0ull, 0ull);
                        if (b < nb) {
                            n = min(cnt_s[b], DHSA_PT_SLOT_CAP);
                            w2 = *reinterpret_cast<const ulonglong2 *>(region + b * DHSA_PT_SLOT_WORDS + 2u * sub);
                            if (sub == 0) w2.x = (unsigned long long)n;
                            if (2u * sub <= n)
                                *reinterpret_cast<ulonglong2 *>(tile_slots + b * DHSA_PT_SLOT_WORDS + 2u * sub) = w2;
                        }
                        __syncwarp();
                        if (b < nb && sub == 0) cnt_s[b] = 0u;
                    }
                    // the overflow list, one packet per thread
                    const uint32_t n_ovf = min(cnt_s[nb], DHSA_PT_OVF);
                    if (n_ovf) {
                        for (uint32_t i = tid; i < n_ovf; i += NPT) {
                            const unsigned long long e = ovf_s[i];
                            pt_update_direct<R>(words, p, wshift, (uint32_t)(e >> 32), (uint32_t)e);
                            direct++;
                        }
                        bar_sync_named(1, NPT);
                        if (tid == 0) cnt_s[nb] = 0u;
                    }
                }
            }
            __threadfence();
            bar_sync_named(1, NPT);
            if (tid == 0) red_release_inc(pp.sync + (c & 3u));
        }
        for (int d = 16; d > 0; d >>= 1) direct += __shfl_xor_sync(0xFFFFFFFFu, direct, d);
        if (lane == 0 && direct) atomicAdd(pp.stats + 2, direct);
        flush_tally(src, on_time, late, lane);
    } else {
        // ------------------------------------------------------------ consumers --
        constexpr int NCT = DHSA_PT_CWARPS * 32;
        const uint32_t cw = warp - DHSA_PT_PWARPS, ctid = tid - DHSA_PT_PWARPS * 32;
        unsigned long long *q = queue_s + cw * DHSA_PT_QUEUE;
        uint32_t qn = 0;
        const uint32_t lt_mask = (1u << lane) - 1u;
        const uint32_t lo32 = lo_s[x];
        uint32_t lookups32 = 0, hits32 = 0, unstored = 0;  // per thread and launch: far below 2^32

        for (uint64_t c = 0; c < nchunks; c++) {
            if (ctid == 0) pt_wait_ge(pp.sync + (c & 3u), nb * (unsigned int)(c / 4 + 1));
            bar_sync_named(2, NCT);
            const uint64_t t0 = c * tiles_per_chunk;
            const uint32_t nt = (uint32_t)(ntiles - t0 < tiles_per_chunk ? ntiles - t0 : tiles_per_chunk);
            const unsigned long long *mine =
                pp.ring + ((c % DHSA_PT_RING) * slots_per_chunk + x) * DHSA_PT_SLOT_WORDS + lane;
            for (uint32_t s = cw; s < nt; s += DHSA_PT_TRIP * DHSA_PT_CWARPS) {
                unsigned long long w[DHSA_PT_TRIP];
#pragma unroll
                for (int u = 0; u < DHSA_PT_TRIP; u++) {
                    const uint32_t su = s + u * DHSA_PT_CWARPS;
                    w[u] = su < nt ? ld_slot_word(mine + (uint64_t)su * nb * DHSA_PT_SLOT_WORDS) : 0ull;
                }
                bool miss[DHSA_PT_TRIP];
#pragma unroll
                for (int u = 0; u < DHSA_PT_TRIP; u++) {
                    const uint32_t n = min((uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)w[u], 0), DHSA_PT_SLOT_CAP);
                    const bool valid = lane >= 1u && lane <= n;
                    const uint32_t set1 = (uint32_t)w[u] & (DHSA_PT_SETS - 1u);
                    const uint32_t tag = (uint32_t)(w[u] >> DHSA_PT_LOG2_SETS);
                    const uint32_t e1 = (tag << 1) + 1u, e2 = e1 + 1u;
                    const uint4 s1 = table[set1];
                    bool hit = s1.x == e1 || s1.y == e1 || s1.z == e1 || s1.w == e1;
                    if (valid && !hit) {
                        const uint32_t set2 = set1 ^ ((tag * 0x9E3779B1u) >> (32 - DHSA_PT_LOG2_SETS));
                        const uint4 s2 = table[set2];
                        hit = s2.x == e2 || s2.y == e2 || s2.z == e2 || s2.w == e2;
                    }
                    miss[u] = valid && !hit;
                    lookups32 += valid;
                    hits32 += valid && hit;
                }
#pragma unroll
                for (int u = 0; u < DHSA_PT_TRIP; u++) {
                    const unsigned bal = __ballot_sync(0xFFFFFFFFu, miss[u]);
                    if (miss[u]) q[qn + __popc(bal & lt_mask)] = w[u];
                    qn += __popc(bal);
                }
                __syncwarp();
                while (qn >= 32u) {
                    qn -= 32u;
                    pt_drain32<R>(words, p, wshift, lo32, table, q + qn, 32u, lane, unstored);
                    __syncwarp();
                }
            }
            bar_sync_named(2, NCT);  // every slot of this chunk has been read into registers
            if (ctid == 0) red_release_inc(pp.sync + 4 + (c & 3u));
        }
        if (qn) pt_drain32<R>(words, p, wshift, lo32, table, q, qn, lane, unstored);
        unsigned long long uns = unstored, lookups = lookups32, hits = hits32;
        for (int d = 16; d > 0; d >>= 1) {
            lookups += __shfl_xor_sync(0xFFFFFFFFu, lookups, d);
            hits += __shfl_xor_sync(0xFFFFFFFFu, hits, d);
            uns += __shfl_xor_sync(0xFFFFFFFFu, uns, d);
        }
        if (lane == 0) {
            if (lookups) atomicAdd(pp.stats + 0, lookups);
            if (hits) atomicAdd(pp.stats + 1, hits);
            if (uns) atomicAdd(pp.stats + 3, uns);
        }
    }
}

}  // namespace dhsa
