// dhsa_device.cuh -- sm_100a kernels of the super point detector hot path.
//
// Written from the algorithm's definition for B200; the reference citations
// (paths relative to /root/reference) say which reference behaviour each kernel
// reproduces bit for bit, not where code came from -- the reference has no GPU
// code at all.
//
// Data layout in HBM
//   bits    r * 2^k cells of g bits, the reference's snapshot layout
//           (pkg/src/dhsa/dhla.py:64-67, estimator.py:3-5).  Kernels view it as
//           little-endian 32-bit words: global bit B = cell * g + b lives at bit
//           B & 31 of word B >> 5, which is bit b % 8 of byte b / 8 of the cell.
//   cand/opp  SoA uint32 packet stream, 8 B per packet, read once.
//
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dhsa {

struct DevParams {
    int r, k, alpha, log2g, key_width;
    uint32_t kmask;  // 2^k - 1
    uint32_t gmask;  // g - 1
    uint64_t state_dh0, state_h1;
    uint64_t ncell;   // r * 2^k
    uint64_t nwords;  // 32-bit words backing the bit array (allocation is padded to 16 B)
    // flow cache (scan mode 3): fc_sets (a power of two) sets of 8 ways x 4 B, one 32-byte sector per set
    unsigned long long *fcache;
    uint32_t fc_sets;
    int fc_shift;                  // 32 - log2(fc_sets): set = a >> fc_shift
    int fc_tag_bits;               // fc_shift + log2(g): key bits an entry stores
    uint32_t fc_epoch;             // entries of other epochs count as empty: a window reset is epoch + 1
    unsigned long long *fc_stats;  // [0] lookups, [1] hits, [2] k_auto_decide's verdict (0 none, 1 cache pays, 2 it does not)
    int gate;                      // scan kernels of a device-gated auto launch: 0 run; 1 run iff k_auto_decide found that
                                   // the flow cache pays in this window; 2 run iff it does not (fc_stats[2], scan_gated_out)
};

// Device-resident control block of one read-out: every stage kernel reads its
// trip counts from here, so the whole chain is stream-ordered with no host sync.
struct Control {
    unsigned long long hot_counts[64];
    unsigned long long stage_counts[64];  // survivors after stage 1, 2, ...
    long long zero_totals[64];            // ZR(i)
    unsigned long long n_candidates;
    unsigned long long n_reports;
    unsigned long long fail_count;
    int fail_stage;
    int flow_saturated;
    int any_empty;  // some hot set is empty -> no candidates (dhla.py:208-209)
    int sorted;     // reports/candidates were sorted on the device by the single-CTA sorter
    unsigned int blocks_done;  // k_hot_sets: CTAs finished (the last one computes the scalars)
    int sz_cut;  // report filter as an integer: a candidate passes iff max(SZ, 1) <= sz_cut (see plan_readout)
    double flow_count, psi, denom;
    unsigned long long counters[4];  // the window's counters as of this read-out: records fed / dropped, flow-cache
                                     // lookups / hits (copied by the chain's last kernel)
};

// ------------------------------------------------------------------ hashing --

// splitmix64 finaliser: pkg/src/dhsa/dhg.py:36-44, pkg/src/dhsa/_core.pyx:35-40.
__device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

// dh0: pkg/src/dhsa/dhg.py:126-128
__device__ __forceinline__ uint32_t dh0_of(const DevParams &p, uint64_t a)
{
    return (uint32_t)mix64(p.state_dh0 ^ a) & p.kmask;
}

// index of key `a` in array i given d0 = dh0(a): pkg/src/dhsa/dhg.py:131-139,152-158
__device__ __forceinline__ uint32_t index_of(const DevParams &p, uint64_t a, uint32_t d0, int i)
{
    return i == 0 ? d0 : (((uint32_t)(a >> ((i - 1) * p.alpha)) & p.kmask) ^ d0);
}

// The dedup key of a packet.  Its R bits depend on (cand, h1(opp)) only (_core.pyx:78-86), so
// both "seen before" tables key on that pair -- 32 + log2(g) bits, 42 at the defaults -- not on
// the 64-bit (cand, opp), and a scanner's thousands of flows collapse to at most g keys.
// a = fmix32(cand ^ h * C) is a bijection of cand for every h (murmur3's 32-bit finaliser), so
// (a, h) still identifies the key: a table indexed by some bits of a only has to store the rest.
#define DHSA_KEY_MUL 0x9E3779B1u

__device__ __forceinline__ uint32_t fmix32(uint32_t a)
{
    a ^= a >> 16;
    a *= 0x85EBCA6Bu;
    a ^= a >> 13;
    a *= 0xC2B2AE35u;
    a ^= a >> 16;
    return a;
}

__device__ __forceinline__ uint32_t unfmix32(uint32_t a)
{
    a ^= a >> 16;
    a *= 0x7ED1B41Du;  // inverse of 0xC2B2AE35 modulo 2^32
    a ^= a >> 13;
    a ^= a >> 26;
    a *= 0xA5CB9243u;  // inverse of 0x85EBCA6B modulo 2^32
    a ^= a >> 16;
    return a;
}

// h1(opp) = mix64(state_h1 ^ opp) & (g - 1) (dhg.py:141-143) with the high word of the first
// two steps folded into per-thread constants: opp only reaches the low word of state_h1 ^ opp.
struct H1Consts {
    uint32_t s_lo, k_shift, m1_hi_term;
};

__device__ __forceinline__ H1Consts h1_consts(uint64_t state_h1)
{
    const uint32_t s_hi = (uint32_t)(state_h1 >> 32);
    H1Consts c;
    c.s_lo = (uint32_t)state_h1;
    c.k_shift = s_hi << 2;                               // bits the first xorshift moves into the low word
    c.m1_hi_term = (s_hi ^ (s_hi >> 30)) * 0x1CE4E5B9u;  // (high word after the xorshift) * low(M1)
    return c;
}

__device__ __forceinline__ uint32_t h1_fast(const H1Consts &c, uint32_t opp, uint32_t gmask)
{
    uint32_t xl = c.s_lo ^ opp;
    xl ^= (xl >> 30) | c.k_shift;                        // z ^= z >> 30, low word
    uint64_t z = (uint64_t)xl * 0x1CE4E5B9u;             // z *= 0xBF58476D1CE4E5B9
    z += (uint64_t)(xl * 0xBF58476Du + c.m1_hi_term) << 32;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    return ((uint32_t)z ^ (uint32_t)(z >> 31)) & gmask;
}

// ---------------------------------------------------------- memory helpers --

// Packet stream: read once, 16 B per lane, kept out of L1 and first in line for
// L2 eviction so it never displaces the sketch.  (On sm_100a the direct
// .L2::evict_first qualifier exists only for 32-byte loads, so the priority is
// passed as a cache-policy operand.)
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint4 *ptr, uint64_t pol)
{
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ptr), "l"(pol));
    return v;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *ptr, uint64_t pol)
{
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(ptr), "l"(pol));
    return v;
}

// Sketch word test-load.  L1 may serve it: bits only ever go 0 -> 1 inside a
// window and L1 is invalidated at every launch, so a stale line can only show a
// set bit as clear, which costs one redundant (idempotent) atomic, never a miss.
__device__ __forceinline__ uint32_t ld_sketch(const uint32_t *ptr)
{
    uint32_t v;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
    return v;
}

// One flow-cache set: 8 ways x 4 B = one 32-byte sector, fetched with a single
// 256-bit load (sm_100a).  Served from L2 only: the table is far larger than L1.
__device__ __forceinline__ void ld_fc_set(const unsigned long long *set, unsigned long long (&e)[4])
{
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(e[0]), "=l"(e[1]), "=l"(e[2]), "=l"(e[3])
                 : "l"(set)
                 : "memory");
}

__device__ __forceinline__ void st_fc_way(uint32_t *slot, uint32_t v)
{
    asm volatile("st.global.cg.u32 [%0], %1;" ::"l"(slot), "r"(v) : "memory");
}

// Fire-and-forget atomic OR (SASS: RED.E.OR), resolved in the L2 slice that owns the word.
__device__ __forceinline__ void red_or(uint32_t *ptr, uint32_t m)
{
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(ptr), "r"(m) : "memory");
}

// --------------------------------------------------------------- K1: scan --
//
// Backend.update_batch (pkg/src/dhsa/_core.pyx:75-86): for each packet, bit
// h1(opp) of cell (i, idx_i(cand)) for every array i.
//
// Fast path: 4 packets per lane per trip (two 16-byte loads), R arrays
// unrolled, 32-bit word addressing (g >= 32, sketch < 16 GiB).  All 4*R test
// loads of a lane are issued before the first is consumed, so each lane keeps
// up to 20 L2 requests in flight.
//
//   MODE 0  one RED per (packet, array), unconditionally
//   MODE 1  test the word first; RED only where the bit is still clear
//           (Alg. 1's "if the bit is 1, continue")
//   MODE 2  as 1, plus warp aggregation: lanes that still need a RED vote,
//           __match_any_sync groups them by word, masks are OR-ed inside a
//           group and its lowest lane issues one RED.
//   (the flow-cache variant, scan mode 3, is k_scan_flowcache below)

// Warp-aggregated RED of one (word, mask) per lane: lanes that need one vote,
// __match_any_sync groups them by word, the group's masks are OR-ed and its
// lowest lane issues a single RED.  Called by all 32 lanes.
__device__ __forceinline__ void red_or_aggregated(uint32_t *words, uint32_t widx, uint32_t mask, bool need,
                                                  uint32_t lane)
{
    const unsigned nm = __ballot_sync(0xFFFFFFFFu, need);
    if (nm == 0) return;  // warp-uniform: nothing new in this slot
    if (need) {
        uint32_t m = mask;
        unsigned peers = 1u << lane;
        if (nm & (nm - 1)) {  // more than one lane: group by word
            peers = __match_any_sync(nm, widx);
            if (peers & (peers - 1)) {  // every member folds every member's mask
                for (unsigned q = peers; q; q &= q - 1) m |= __shfl_sync(peers, mask, __ffs(q) - 1);
            }
        }
        if (lane == (uint32_t)(__ffs(peers) - 1)) red_or(words + widx, m);
    }
}

template <int R>
__device__ __forceinline__ void packet_slots(const DevParams &p, int wshift, uint32_t cand, uint32_t h, uint32_t d0,
                                             uint32_t (&widx)[R])
{
    const uint32_t hw = h >> 5;
#pragma unroll
    for (int i = 0; i < R; i++) {
        const uint32_t idx = i == 0 ? d0 : (((uint32_t)((uint64_t)cand >> ((i - 1) * p.alpha)) & p.kmask) ^ d0);
        const uint32_t cell = ((uint32_t)i << p.k) | idx;
        widx[i] = (cell << wshift) + hw;
    }
}

// ------------------------------------------- TMA bulk copies + mbarriers --
// cp.async.bulk (SASS UBLKCP): the TMA engine moves a contiguous run of global
// memory into shared memory and signals an mbarrier with the byte count, so the
// packet stream neither occupies registers nor competes with the scattered
// sketch / flow-cache accesses for the SM's L1-miss request port.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t arrivals)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(arrivals) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(mbar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t smem_dst, const void *gmem_src, uint32_t bytes, uint32_t mbar,
                                         uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_dst),
        "l"(gmem_src), "r"(bytes), "r"(mbar), "l"(pol)
        : "memory");
}

// order this thread's earlier generic-proxy accesses to shared memory before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------- packet sources --
// Where a lane's 4 packets per trip come from.  The scan kernels are templated
// on the source, so decode is fused into the scan instead of being a pass.
//
//   SoaSource     the reference's batch form: uint32 cand[], opp[] (8 B per packet),
//                 Backend.update_batch(cand, opp) -- pkg/src/dhsa/_core.pyx:52-59.
//   RecordSource  raw 12-byte IPPR trace records -- u32 timestamp little-endian, src
//                 and dst IPv4 as u32 big-endian (pkg/src/dhsa/ingest.py:20) -- with
//                 the window engine's per-record work folded in: window id =
//                 ts // window_seconds (engine.py:140), late-record drop
//                 (wins == arrival, engine.py:148), direction policy
//                 (split_pairs, engine.py:179-194; "both" is two launches).
//                 4 records = 48 B = three 16-byte loads per lane.
struct SoaSource {
    const uint4 *cand4, *opp4;
    uint64_t nvec;
    static constexpr bool kTally = false;
    struct Raw {
        uint4 c, o;
    };
    __host__ __device__ __forceinline__ uint64_t vectors() const { return nvec; }
    __device__ __forceinline__ void load(Raw &r, uint64_t v, uint64_t pol) const
    {
        r.c = make_uint4(0, 0, 0, 0), r.o = make_uint4(0, 0, 0, 0);
        if (v < nvec) {
            r.c = ld_stream_v4(cand4 + v, pol);
            r.o = ld_stream_v4(opp4 + v, pol);
        }
    }
    // staged form: one stage = kTrips warp trips = kTrips * 32 vectors of cand, then as many of opp, in shared
    // memory; one mbarrier wait, one refill (two bulk copies) per stage
#ifndef DHSA_FC_SOA_TRIPS
#define DHSA_FC_SOA_TRIPS 4
#endif
#ifndef DHSA_FC_SOA_STAGES
#define DHSA_FC_SOA_STAGES 2
#endif
#ifndef DHSA_FC_TRIP_UNROLL
#define DHSA_FC_TRIP_UNROLL 1
#endif
#define DHSA_STR_(x) #x
#define DHSA_UNROLL(n) _Pragma(DHSA_STR_(unroll n))
    static constexpr int kTrips = DHSA_FC_SOA_TRIPS;
    static constexpr int kStageBytes = 1024 * kTrips;
    static constexpr int kStages = DHSA_FC_SOA_STAGES;
    __device__ __forceinline__ void stage_issue(uint32_t smem_dst, uint32_t mbar, uint64_t base, uint32_t count,
                                                uint64_t pol) const
    {
        const uint32_t bytes = count * 16u;
        mbar_expect_tx(mbar, 2u * bytes);
        bulk_g2s(smem_dst, cand4 + base, bytes, mbar, pol);
        bulk_g2s(smem_dst + 512u * kTrips, opp4 + base, bytes, mbar, pol);
    }
    __device__ __forceinline__ void stage_read(Raw &r, const uint8_t *stage, uint32_t idx) const
    {
        r.c = *reinterpret_cast<const uint4 *>(stage + idx * 16u);
        r.o = *reinterpret_cast<const uint4 *>(stage + 512u * kTrips + idx * 16u);
    }
    __device__ __forceinline__ void unpack(const Raw &r, uint64_t v, uint32_t (&cs)[4], uint32_t (&os)[4],
                                           bool (&ok)[4], uint32_t &, uint32_t &) const
    {
        cs[0] = r.c.x, cs[1] = r.c.y, cs[2] = r.c.z, cs[3] = r.c.w;
        os[0] = r.o.x, os[1] = r.o.y, os[2] = r.o.z, os[3] = r.o.w;
        ok[0] = ok[1] = ok[2] = ok[3] = v < nvec;
    }
};

struct RecordSource {
    const uint4 *rec4;        // quad q (records first_rec + 4q .. + 3) = rec4[3q .. 3q + 2]
    uint64_t nquads;
    uint64_t first_rec;       // record index of quad 0 in the caller's stream
    uint64_t rec_lo, rec_hi;  // records of this launch: one window's contiguous segment
    uint32_t window_seconds;
    uint32_t window_id;
    uint32_t ts_lo, ts_hi;    // timestamps of this window, inclusive (set_window)
    int cand_is_dst;          // direction policy: 0 "src" (cand = src), 1 "dst" (cand = dst)
    unsigned long long *tally;  // [0] pairs fed (on-time records), [1] late records dropped
    int tally_late;             // 0 on the second pass of "both", so a late record is counted once
    static constexpr bool kTally = true;
    struct Raw {
        uint4 a, b, c;
    };
    // timestamps with ts // seconds == id, clamped to 32 bits; seconds == 0 takes every record
    __host__ void set_window(uint32_t seconds, uint32_t id)
    {
        window_seconds = seconds, window_id = id;
        const unsigned long long lo = (unsigned long long)seconds * id, hi = lo + seconds - 1ull;
        ts_lo = seconds == 0u ? 0u : (lo > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)lo);
        ts_hi = seconds == 0u ? 0xFFFFFFFFu : (hi > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)hi);
        if (seconds != 0u && lo > 0xFFFFFFFFull) ts_lo = 1u, ts_hi = 0u;  // window beyond any 32-bit timestamp: empty
    }
    __host__ __device__ __forceinline__ uint64_t vectors() const { return nquads; }
    __device__ __forceinline__ void load(Raw &r, uint64_t v, uint64_t pol) const
    {
        r.a = r.b = r.c = make_uint4(0, 0, 0, 0);
        if (v < nquads) {
            r.a = ld_stream_v4(rec4 + 3 * v + 0, pol);
            r.b = ld_stream_v4(rec4 + 3 * v + 1, pol);
            r.c = ld_stream_v4(rec4 + 3 * v + 2, pol);
        }
    }
    // staged form: one warp trip = 32 quads = 1536 contiguous bytes of records; kTrips trips per stage
#ifndef DHSA_FC_REC_TRIPS
#define DHSA_FC_REC_TRIPS 2
#endif
#ifndef DHSA_FC_REC_STAGES
#define DHSA_FC_REC_STAGES 2
#endif
    static constexpr int kTrips = DHSA_FC_REC_TRIPS;
    static constexpr int kStageBytes = 1536 * kTrips;
    static constexpr int kStages = DHSA_FC_REC_STAGES;
    __device__ __forceinline__ void stage_issue(uint32_t smem_dst, uint32_t mbar, uint64_t base, uint32_t count,
                                                uint64_t pol) const
    {
        const uint32_t bytes = count * 48u;
        mbar_expect_tx(mbar, bytes);
        bulk_g2s(smem_dst, rec4 + 3 * base, bytes, mbar, pol);
    }
    __device__ __forceinline__ void stage_read(Raw &r, const uint8_t *stage, uint32_t idx) const
    {
        const uint4 *q = reinterpret_cast<const uint4 *>(stage + idx * 48u);
        r.a = q[0], r.b = q[1], r.c = q[2];
    }
    __device__ __forceinline__ void unpack(const Raw &r, uint64_t v, uint32_t (&cs)[4], uint32_t (&os)[4],
                                           bool (&ok)[4], uint32_t &on_time, uint32_t &late) const
    {
        const uint32_t w[12] = {r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w, r.c.x, r.c.y, r.c.z, r.c.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint64_t idx = first_rec + 4 * v + (uint64_t)j;
            const bool mine = v < nquads && idx >= rec_lo && idx < rec_hi;
            const uint32_t ts = w[3 * j];
            const uint32_t src = __byte_perm(w[3 * j + 1], 0, 0x0123);  // network order -> host order
            const uint32_t dst = __byte_perm(w[3 * j + 2], 0, 0x0123);
            // ts // window_seconds == window_id as a range test (no division): [ts_lo, ts_hi] was set by the host.
            // window_seconds == 0: no windowing, every record of the range is taken (exact oracle over a whole trace)
            const bool fresh = mine && ts >= ts_lo && ts <= ts_hi;
            cs[j] = cand_is_dst ? dst : src;
            os[j] = cand_is_dst ? src : dst;
            ok[j] = fresh;
            on_time += fresh;
            late += mine && !fresh && tally_late;
        }
    }
};

template <typename SRC>
__device__ __forceinline__ void flush_tally(const SRC &src, uint32_t on_time, uint32_t late, uint32_t lane)
{
    if (!SRC::kTally) return;
    for (int d = 16; d > 0; d >>= 1) {
        on_time += __shfl_xor_sync(0xFFFFFFFFu, on_time, d);
        late += __shfl_xor_sync(0xFFFFFFFFu, late, d);
    }
    if (lane == 0) {
        if (on_time) atomicAdd(((const RecordSource &)src).tally + 0, (unsigned long long)on_time);
        if (late) atomicAdd(((const RecordSource &)src).tally + 1, (unsigned long long)late);
    }
}

// Scan mode `auto`, decided on the device.  A window starts behind the flow cache; whether the cache pays (flows repeat)
// is known only from its own counters.  Between launches the host reads them (dhsa_cabi.cu: the auto policy); for ONE long
// launch it queues four kernels: the first DHSA_GATE_SAMPLE packets through the cache, k_auto_decide, then the rest
// through the test-first kernel with gate = 2 and through the cache kernel with gate = 1.  Exactly one of the two does
// the work; the other returns at once (scan_gated_out).
//
// The verdict must not be fooled by a cold table: the first m packets of a window over F equally likely flows find only
// ~m/2F of their keys, however often the flows will repeat later (config 2: 13% hits in the first million packets, 96%
// over the window).  So the sample's counts are projected: with D = m - hits distinct keys among m lookups,
// x = m / F solves (1 - e^-x) / x = D / m, and over the N = m + rest packets of this launch the same population would
// miss (1 - e^-y) / y of its lookups, y = x N / m.  The cache pays when that projected miss rate is at most 0.7 --
// the host policy's break-even (1 + 11 (1 - h) requests per packet with the cache, 5 + 5 (1 - h) without).
#define DHSA_POLICY_MIN_SAMPLE (1ull << 22)
#define DHSA_GATE_SAMPLE (1ull << 20)
__global__ void k_auto_decide(unsigned long long *fc_stats, unsigned long long rest_packets)
{
    const unsigned long long m = fc_stats[0], h = fc_stats[1];
    bool pays = true;
    if (m > 0) {
        const float rho = (float)(m - h) / (float)m;
        float lo = 1e-7f, hi = 64.0f;  // (1 - e^-x) / x falls from 1 to 0
        for (int it = 0; it < 28; it++) {  // fp32: 28 halvings of [1e-7, 64] are below its resolution
            const float x = 0.5f * (lo + hi);
            if (-expm1f(-x) / x > rho) lo = x; else hi = x;
        }
        const float y = 0.5f * (lo + hi) * ((float)m + (float)rest_packets) / (float)m;
        pays = -expm1f(-y) / y <= 0.7f;
    }
    fc_stats[2] = pays ? 1ull : 2ull;
}

__device__ __forceinline__ bool scan_gated_out(const DevParams &p)
{
    if (p.gate == 0) return false;
    const bool no_repeats = p.fc_stats[2] == 2ull;
    return (p.gate == 1) == no_repeats;
}

// GATED: the instantiation a device-gated auto launch uses (it first asks scan_gated_out).  The plain instantiations
// do not contain the check at all: with it in the prologue nvcc scheduled the flow-cache kernel's lookup loop
// differently (+4% instructions, scan 0.548 -> 0.568 ms).
template <int R, int MODE, typename SRC, bool GATED = false>
__global__ void __launch_bounds__(256) k_scan_vec4(SRC src, uint32_t *__restrict__ words, DevParams p)
{
    if (GATED && scan_gated_out(p)) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nvec = src.vectors();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int wshift = p.log2g - 5;
    const uint64_t pol = policy_evict_first();
    uint32_t on_time = 0, late = 0;

    for (uint64_t base = warp0 * 32; base < nvec; base += nwarps * 32) {
        const uint64_t v = base + lane;
        typename SRC::Raw raw;
        src.load(raw, v, pol);
        uint32_t cs[4], os[4];
        bool ok[4];
        src.unpack(raw, v, cs, os, ok, on_time, late);

        uint32_t widx[4][R];
        uint32_t mask[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t h = (uint32_t)mix64(p.state_h1 ^ (uint64_t)os[j]) & p.gmask;
            const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ (uint64_t)cs[j]) & p.kmask;
            mask[j] = 1u << (h & 31u);
            packet_slots<R>(p, wshift, cs[j], h, d0, widx[j]);
        }
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (ok[j]) {
#pragma unroll
                    for (int i = 0; i < R; i++) red_or(words + widx[j][i], mask[j]);
                }
        } else {
            // all 4 * R test loads are issued before the first is consumed
            uint32_t w[4][R];
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int i = 0; i < R; i++) w[j][i] = ok[j] ? ld_sketch(words + widx[j][i]) : 0xFFFFFFFFu;
#pragma unroll
            for (int j = 0; j < 4; j++) {
#pragma unroll
                for (int i = 0; i < R; i++) {
                    const bool need = (w[j][i] & mask[j]) == 0;
                    if (MODE == 1) {
                        if (need) red_or(words + widx[j][i], mask[j]);
                    } else {
                        red_or_aggregated(words, widx[j][i], mask[j], need, lane);
                    }
                }
            }
        }
    }
    flush_tally(src, on_time, late, lane);
}

// K1, scan mode 3: the scan behind an exact flow cache.
//
// ncu shows k_scan_vec4 pinned at one L1-miss request per clock per SM
// (l1tex__m_l1tex2xbar_req_cycles_active 92%) with 5 sketch sectors per packet,
// so the lever is fewer scattered accesses per packet.  Real windows carry many
// packets per flow (BASELINE config 2: ~26), and a repeated key changes nothing
// in the sketch.  The cache is an 8-way set-associative table of keys in L2, one
// 32-byte sector per set, read with a single 256-bit load: a packet whose key is
// present was scanned earlier in this window and is dropped after ONE scattered
// access instead of five.
//
//   key        (cand, h = h1(opp)), see fmix32 above.  set = top bits of
//              a = fmix32(cand ^ h * C); the entry is the rest of (a, h) under the
//              table's current epoch (>= 1; entries of other epochs are empty ways, so
//              a window reset is epoch + 1, not a memset): 32 bits instead of the 64-bit pair, so the same number of
//              keys needs half the L2 -- ncu showed a third of the lookups of a 64 MiB
//              pair table served from HBM -- and a set holds 8 ways instead of 4.
//              (set, entry) determines (a, h), hence (cand, h): a hit is never another key.
//   exactness  an entry is written only by a lane that has just issued the
//              key's own test+RED, the table is cleared whenever bits can
//              disappear (reset, upload), and nothing reads bits before the
//              kernel ends -- so "present => bits set at kernel end" always holds
//              and a missing / racing entry only costs a rescan.
//   misses     are compacted by ballot into a per-warp shared-memory queue and
//              drained 32 at a time, one missed packet per lane with its R test
//              loads in flight together, so a miss costs one more L2 round trip
//              per 32 misses, not per packet slot.
//   pipeline   the packet stream is staged by TMA, several trips ahead.

#define DHSA_FC_NO_SLOT 0xFFFFFFFFu
#ifndef DHSA_FC_SKIP_TEST
#define DHSA_FC_SKIP_TEST 1
#endif
#ifndef DHSA_FC_CTAS_PER_SM
#define DHSA_FC_CTAS_PER_SM 3
#endif
// A queued miss is just the key.  Everything only a miss needs -- the empty-way search, dh0, the R
// word indices -- happens in the drain, where all 32 lanes hold a miss: in the lookup loop the same
// code ran under `if (miss)` with one or two active lanes per warp (4% of the packets miss, so three
// packet slots in four have at least one) and cost 7% of the kernel's instructions.  The drain
// re-reads the key's set (one more L2 sector per miss, +3% requests): it needs the ways to pick the
// slot, and a key another warp recorded in the meantime turns into a hit there (-20% REDs).
struct FcMiss {
    uint32_t cand, h;
};

// (set, entry) of a key in a table of 2^(32 - shift) sets
__device__ __forceinline__ void fc_locate(const DevParams &p, uint32_t cand, uint32_t h, uint32_t &set, uint32_t &entry)
{
    const uint32_t a = fmix32(cand ^ (h * DHSA_KEY_MUL));
    set = a >> p.fc_shift;
    entry = (p.fc_epoch << p.fc_tag_bits) | ((a & ((1u << p.fc_shift) - 1u)) << p.log2g) | h;  // epoch >= 1
}

// The way of set `set_idx` a new key goes to: the first empty way (an entry of another epoch) as
// loaded, searched from a key-dependent start so that lanes which loaded the same still-empty set do
// not all pick way 0 and overwrite each other; DHSA_FC_NO_SLOT when the set is full (no eviction:
// evicting a live key only moves the miss to another key and costs a store; the table empties with
// every window).  A race only loses an entry.
__device__ __forceinline__ uint32_t fc_pick_slot(const DevParams &p, const uint32_t (&way)[8], uint32_t set_idx,
                                                 uint32_t entry)
{
    uint32_t empty = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) empty |= (uint32_t)((way[t] >> p.fc_tag_bits) != p.fc_epoch) << t;
    const uint32_t rot = entry & 7u;
    const uint32_t turned = ((empty >> rot) | (empty << (8u - rot))) & 0xFFu;
    return turned ? ((set_idx << 3) | (((uint32_t)(__ffs(turned) - 1) + rot) & 7u)) : DHSA_FC_NO_SLOT;
}

// Drain up to 32 queued misses, one per lane: the R test loads of a lane are in flight
// together, then its REDs, then the key is recorded in the table.
template <int R>
__device__ __forceinline__ void fc_drain32(uint32_t *__restrict__ words, const DevParams &p, int wshift,
                                           const FcMiss *q, uint32_t n_active, uint32_t lane)
{
    bool act = lane < n_active;
    FcMiss m = {0u, 0u};
    if (act) m = q[lane];
    uint32_t set, entry;
    fc_locate(p, m.cand, m.h, set, entry);
    unsigned long long e[4] = {0ull, 0ull, 0ull, 0ull};
    if (act) ld_fc_set(p.fcache + ((size_t)set << 2), e);
    uint32_t way[8];
#pragma unroll
    for (int t = 0; t < 4; t++) way[2 * t] = (uint32_t)e[t], way[2 * t + 1] = (uint32_t)(e[t] >> 32);
    bool hit = false;
#pragma unroll
    for (int t = 0; t < 8; t++) hit |= way[t] == entry;
    act = act && !hit;  // recorded by another warp since the lookup: that warp issued its REDs
    const uint32_t slot = fc_pick_slot(p, way, set, entry);
    const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ (uint64_t)m.cand) & p.kmask;
    const uint32_t mask = 1u << (m.h & 31u);
    uint32_t widx[R], w[R];
    packet_slots<R>(p, wshift, m.cand, m.h, d0, widx);
    // A key that found an empty way in its set was never recorded in this window (sets are never
    // evicted), so it is almost surely new and its bits still clear: skip the test loads and RED
    // unconditionally (a RED costs ~1.5 loads in L2, a test that finds the bit clear costs both).
    // Keys from full sets are usually repeats whose bits are set: those test first.
    const bool fresh = DHSA_FC_SKIP_TEST && slot != DHSA_FC_NO_SLOT;
#pragma unroll
    for (int i = 0; i < R; i++) w[i] = act ? (fresh ? 0u : ld_sketch(words + widx[i])) : 0xFFFFFFFFu;
    // Plain REDs, no warp aggregation: every drained key is new to the table and sets its own bit, so a word sees at
    // most 32 REDs (plus lost-race duplicates) per window -- there is no same-address burst to merge, and five
    // MATCH.ANY + shuffle rounds per drain were 10% of the kernel's stall samples.
#pragma unroll
    for (int i = 0; i < R; i++)
        if ((w[i] & mask) == 0) red_or(words + widx[i], mask);
    // the key now counts as scanned: its tests/REDs above are issued before this store
    if (act && slot != DHSA_FC_NO_SLOT) st_fc_way(reinterpret_cast<uint32_t *>(p.fcache) + slot, entry);
}

template <typename SRC>
struct FcSmem {
    static constexpr int kStageBytesAll = 8 * SRC::kStages * SRC::kStageBytes;
    static constexpr int kMbarBytesAll = 8 * SRC::kStages * 8;
    static constexpr int kQueueBytesAll = 8 * (32 + 128) * (int)sizeof(FcMiss);
    static constexpr int kBytes = kStageBytesAll + kMbarBytesAll + kQueueBytesAll;
};

// The packet stream is staged by TMA: every warp owns a ring of SRC::kStages
// shared-memory slots and one mbarrier per slot; lane 0 keeps the ring full with
// cp.async.bulk copies (one warp trip per slot), all lanes wait on the slot's
// mbarrier parity and read their 16-byte vectors with LDS.128.
template <int R, typename SRC, bool GATED = false>
__global__ void __launch_bounds__(256, DHSA_FC_CTAS_PER_SM) k_scan_flowcache(SRC src, uint32_t *__restrict__ words, DevParams p)
{
    if (GATED && scan_gated_out(p)) return;
    // dynamic shared memory (FcSmem<SRC>::kBytes): per-warp stage rings, mbarriers, miss queues
    extern __shared__ __align__(128) uint8_t fc_smem[];
    typedef uint8_t StageRing[SRC::kStages][SRC::kStageBytes];
    StageRing *stage_s = reinterpret_cast<StageRing *>(fc_smem);
    typedef unsigned long long MbarRing[SRC::kStages];
    MbarRing *mbar_s = reinterpret_cast<MbarRing *>(fc_smem + FcSmem<SRC>::kStageBytesAll);
    typedef FcMiss MissQueue[32 + 128];
    MissQueue *queue_s = reinterpret_cast<MissQueue *>(fc_smem + FcSmem<SRC>::kStageBytesAll + FcSmem<SRC>::kMbarBytesAll);
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    FcMiss *q = queue_s[wib];
    uint32_t qn = 0;
    const uint64_t nvec = src.vectors();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    constexpr uint32_t kPerStage = 32u * SRC::kTrips;  // vectors a warp takes per stage
    const uint64_t step = nwarps * kPerStage;
    const int wshift = p.log2g - 5;
    const uint64_t pol = policy_evict_first();
    const uint32_t lt_mask = (1u << lane) - 1u;
    const H1Consts hc = h1_consts(p.state_h1);
    uint32_t fc_miss = 0, fc_trips = 0;  // per thread and launch: far below 2^32
    uint32_t on_time = 0, late = 0;
    // this warp's stage ring and mbarriers as shared-window addresses
    const uint32_t ring_a = smem_u32(stage_s[wib][0]);
    const uint32_t mbar_a = smem_u32(&mbar_s[wib][0]);

    if (lane == 0) {
        for (int st = 0; st < SRC::kStages; st++) mbar_init(mbar_a + 8u * st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // fill the ring
    uint64_t issue_base = warp0 * kPerStage;
    if (lane == 0) {
        for (int st = 0; st < SRC::kStages; st++) {
            if (issue_base < nvec) {
                const uint64_t left = nvec - issue_base;
                src.stage_issue(ring_a + (uint32_t)SRC::kStageBytes * st, mbar_a + 8u * st, issue_base,
                                (uint32_t)(left < kPerStage ? left : kPerStage), pol);
            }
            issue_base += step;
        }
    }
    uint32_t slot = 0, parity = 0;
    for (uint64_t sbase = warp0 * kPerStage; sbase < nvec; sbase += step) {
        mbar_wait(mbar_a + 8u * slot, parity);
      DHSA_UNROLL(DHSA_FC_TRIP_UNROLL)
      for (int tr = 0; tr < SRC::kTrips; tr++) {
        const uint64_t base = sbase + 32u * tr;
        if (base >= nvec) break;  // warp-uniform
        typename SRC::Raw raw;
        src.stage_read(raw, stage_s[wib][slot], lane + 32u * tr);
        if (tr + 1 == SRC::kTrips || base + 32u >= nvec) {  // the stage's last trip has been read: refill the slot
            __syncwarp();
            if (lane == 0) {
                const uint64_t nb = sbase + (uint64_t)SRC::kStages * step;
                if (nb < nvec) {
                    fence_proxy_async_smem();
                    const uint64_t left = nvec - nb;
                    src.stage_issue(ring_a + (uint32_t)SRC::kStageBytes * slot, mbar_a + 8u * slot, nb,
                                    (uint32_t)(left < kPerStage ? left : kPerStage), pol);
                }
            }
            if (++slot == SRC::kStages) {
                slot = 0;
                parity ^= 1u;
            }
        }
        uint32_t cs[4], os[4];
        bool ok[4];
        src.unpack(raw, base + lane, cs, os, ok, on_time, late);
        fc_trips += base + lane < nvec;

        unsigned long long e[4][4];
        uint32_t set_idx[4], entry[4], hs[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            hs[j] = h1_fast(hc, os[j], p.gmask);
            fc_locate(p, cs[j], hs[j], set_idx[j], entry[j]);
            if (ok[j]) ld_fc_set(p.fcache + ((size_t)set_idx[j] << 2), e[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            uint32_t way[8];
#pragma unroll
            for (int t = 0; t < 4; t++) way[2 * t] = (uint32_t)e[j][t], way[2 * t + 1] = (uint32_t)(e[j][t] >> 32);
            bool hit = false;
#pragma unroll
            for (int t = 0; t < 8; t++) hit |= way[t] == entry[j];
            const bool miss = ok[j] && !hit;
            fc_miss += miss;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, miss);
            if (bal == 0) continue;
            if (miss) {
                const FcMiss m = {cs[j], hs[j]};
                q[qn + __popc(bal & lt_mask)] = m;
            }
            qn += __popc(bal);
        }
        __syncwarp();
        while (qn >= 32) {  // dense drains: the newest 32 entries, one per lane
            qn -= 32;
            fc_drain32<R>(words, p, wshift, q + qn, 32, lane);
        }
        __syncwarp();
      }
    }
    if (qn) fc_drain32<R>(words, p, wshift, q, qn, lane);
    // lookups = the packets this lane examined (on-time records of a record source: unpack counted them; every packet
    // of its vectors otherwise), hits = lookups - misses
    unsigned long long lookups64 = SRC::kTally ? on_time : 4u * fc_trips;
    unsigned long long hits64 = lookups64 - fc_miss;
    for (int d = 16; d > 0; d >>= 1) {
        hits64 += __shfl_xor_sync(0xFFFFFFFFu, hits64, d);
        lookups64 += __shfl_xor_sync(0xFFFFFFFFu, lookups64, d);
    }
    if (lane == 0 && lookups64) {
        atomicAdd(p.fc_stats + 0, lookups64);
        atomicAdd(p.fc_stats + 1, hits64);
    }
    flush_tally(src, on_time, late, lane);
}

// General path: any r <= 64, any g >= 8 (sub-word cells included), 64-bit bit
// addressing, unaligned input pointers.  One packet per lane per trip.
template <int MODE>
__global__ void __launch_bounds__(256) k_scan_generic(const uint32_t *__restrict__ cand,
                                                      const uint32_t *__restrict__ opp, uint64_t n,
                                                      uint32_t *__restrict__ words, DevParams p)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t pol = policy_evict_first();
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint64_t a = ld_stream_u32(cand + t, pol);
        const uint64_t h = mix64(p.state_h1 ^ (uint64_t)ld_stream_u32(opp + t, pol)) & p.gmask;
        const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ a) & p.kmask;
        for (int i = 0; i < p.r; i++) {
            const uint64_t cell = ((uint64_t)i << p.k) | index_of(p, a, d0, i);
            const uint64_t B = (cell << p.log2g) + h;
            uint32_t *wp = words + (B >> 5);
            const uint32_t m = 1u << (uint32_t)(B & 31);
            if (MODE == 0 || (ld_sketch(wp) & m) == 0) red_or(wp, m);
        }
    }
}

// Records through the general path (any parameters, ragged ends of a segment):
// one record per lane per trip, 4-byte loads.
template <int MODE>
__global__ void __launch_bounds__(256) k_scan_records_generic(const uint32_t *__restrict__ rec_words, uint64_t rec_lo,
                                                              uint64_t rec_hi, uint32_t window_seconds,
                                                              uint32_t window_id, int cand_is_dst,
                                                              unsigned long long *tally, int tally_late,
                                                              uint32_t *__restrict__ words, DevParams p)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t pol = policy_evict_first();
    uint32_t on_time = 0, late = 0;
    for (uint64_t t = rec_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rec_hi; t += stride) {
        const uint32_t ts = ld_stream_u32(rec_words + 3 * t, pol);
        const uint32_t src = __byte_perm(ld_stream_u32(rec_words + 3 * t + 1, pol), 0, 0x0123);
        const uint32_t dst = __byte_perm(ld_stream_u32(rec_words + 3 * t + 2, pol), 0, 0x0123);
        if (ts / window_seconds != window_id) {
            late += tally_late;
            continue;
        }
        on_time++;
        const uint64_t a = cand_is_dst ? dst : src;
        const uint64_t h = mix64(p.state_h1 ^ (uint64_t)(cand_is_dst ? src : dst)) & p.gmask;
        const uint32_t d0 = (uint32_t)mix64(p.state_dh0 ^ a) & p.kmask;
        for (int i = 0; i < p.r; i++) {
            const uint64_t cell = ((uint64_t)i << p.k) | index_of(p, a, d0, i);
            const uint64_t B = (cell << p.log2g) + h;
            uint32_t *wp = words + (B >> 5);
            const uint32_t m = 1u << (uint32_t)(B & 31);
            if (MODE == 0 || (ld_sketch(wp) & m) == 0) red_or(wp, m);
        }
    }
    if (on_time) atomicAdd(tally + 0, (unsigned long long)on_time);
    if (late) atomicAdd(tally + 1, (unsigned long long)late);
}

// Window plan of a record stream (engine.py:140-149): a record arrives during the
// running maximum of the window ids seen so far, so the stream splits into
// contiguous segments, one per window, at the records where that running maximum
// rises.  Pass 1: per-block maximum window id.  Pass 2 (one CTA): exclusive
// prefix maximum over blocks, seeded with the window already open.  Pass 3:
// every block replays its records against its carry-in and appends a
// (position, new window id) boundary wherever the running maximum rises.
#define DHSA_PLAN_BLOCK 4096  // records per plan block (256 threads x 16)

__global__ void __launch_bounds__(256) k_plan_blockmax(const uint32_t *__restrict__ rec_words, uint64_t n,
                                                       uint32_t window_seconds, uint32_t *__restrict__ block_max)
{
    __shared__ uint32_t warp_max[8];
    const uint64_t lo = (uint64_t)blockIdx.x * DHSA_PLAN_BLOCK;
    uint32_t m = 0;  // floor division is monotone: max(ts) // w == max(ts // w), so divide once per block
    for (uint32_t q = threadIdx.x; q < DHSA_PLAN_BLOCK; q += 256) {
        const uint64_t t = lo + q;
        if (t < n) m = max(m, rec_words[3 * t]);
    }
    for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, d));
    if ((threadIdx.x & 31) == 0) warp_max[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; w++) m = max(m, warp_max[w]);
        block_max[blockIdx.x] = m / window_seconds;
    }
}

// carry[b] = max(seed, block_max[0 .. b-1]) as a signed 64-bit value (seed -1 = no window open yet),
// and the list of blocks in which the running maximum rises (the only ones pass 3 has to read).
// One CTA: every thread takes a contiguous run of blocks, the runs' maxima are scanned across the CTA.
__global__ void __launch_bounds__(1024) k_plan_carry(const uint32_t *__restrict__ block_max, uint64_t nblocks,
                                                     long long seed, long long *__restrict__ carry,
                                                     uint32_t *__restrict__ rise_list, unsigned int *__restrict__ rise_count)
{
    __shared__ long long warp_tot[32];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const uint64_t per = (nblocks + 1023) / 1024;
    const uint64_t lo = min((uint64_t)threadIdx.x * per, nblocks), hi = min(lo + per, nblocks);
    long long local = -1;
    for (uint64_t b = lo; b < hi; b++) local = max(local, (long long)block_max[b]);
    long long inc = local;
    for (int d = 1; d < 32; d <<= 1) {
        const long long t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= (uint32_t)d) inc = max(inc, t);
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    long long run = seed;
    for (uint32_t w = 0; w < wid; w++) run = max(run, warp_tot[w]);
    long long excl = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
    if (lane == 0) excl = -1;
    run = max(run, excl);
    for (uint64_t b = lo; b < hi; b++) {
        const long long mine = (long long)block_max[b];
        carry[b] = run;
        if (mine > run) {
            rise_list[atomicAdd(rise_count, 1u)] = (uint32_t)b;
            run = mine;
        }
    }
}

struct PlanBoundary {
    unsigned long long position;  // first record of the segment
    long long window_id;
};

__global__ void __launch_bounds__(256) k_plan_boundaries(const uint32_t *__restrict__ rec_words, uint64_t n,
                                                         uint32_t window_seconds,
                                                         const long long *__restrict__ carry,
                                                         const uint32_t *__restrict__ rise_list,
                                                         const unsigned int *__restrict__ rise_count,
                                                         PlanBoundary *__restrict__ out, unsigned int cap,
                                                         unsigned int *__restrict__ count)
{
    // only blocks in which the running maximum rises are visited (a handful per chunk of a
    // time-ordered trace).  256 threads x 16 consecutive records: thread-local running max, block
    // scan of the per-thread maxima, then each thread replays its 16 records against its own carry-in
    __shared__ long long warp_tot[8];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const unsigned int n_rise = *rise_count;
    for (unsigned int r = blockIdx.x; r < n_rise; r += gridDim.x) {
        const uint32_t blk = rise_list[r];
        const uint64_t t0 = (uint64_t)blk * DHSA_PLAN_BLOCK + (uint64_t)threadIdx.x * 16;
        long long win[16];
        long long tmax = -1;
#pragma unroll
        for (int q = 0; q < 16; q++) {
            win[q] = t0 + q < n ? (long long)(rec_words[3 * (t0 + q)] / window_seconds) : -1;
            tmax = max(tmax, win[q]);
        }
        long long inc = tmax;
        for (int d = 1; d < 32; d <<= 1) {
            const long long t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= (uint32_t)d) inc = max(inc, t);
        }
        if (lane == 31) warp_tot[wid] = inc;
        __syncthreads();
        long long run = carry[blk];
        for (uint32_t w = 0; w < wid; w++) run = max(run, warp_tot[w]);
        long long excl = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
        if (lane == 0) excl = -1;
        run = max(run, excl);
#pragma unroll
        for (int q = 0; q < 16; q++) {
            if (win[q] > run) {
                run = win[q];
                const unsigned int pos = atomicAdd(count, 1u);
                if (pos < cap) {
                    out[pos].position = t0 + q;
                    out[pos].window_id = run;
                }
            }
        }
        __syncthreads();  // warp_tot is reused by the next block of this CTA
    }
}

// ------------------------------------------------- K2: per-cell estimation --
//
// Backend.zero_counts (pkg/src/dhsa/_core.pyx:89-118): zc = g - popcount(cell).
// LANES lanes cooperate on one cell, each popcounting 16-byte vectors, so a
// warp reads 512 contiguous bytes per step at g = 1024 (4 cells per warp).
__global__ void __launch_bounds__(256) k_zero_counts_vec(const uint4 *__restrict__ bits16,
                                                         int32_t *__restrict__ zc, uint64_t ncell,
                                                         int vecs_per_cell, int lanes, int g)
{
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t cells_per_pass = ((uint64_t)gridDim.x * blockDim.x) / (uint64_t)lanes;
    const uint32_t sub = (uint32_t)(gtid % (uint64_t)lanes);
    // every lane runs the same number of passes (the shuffles below need full warps)
    for (uint64_t cell0 = 0; cell0 < ncell; cell0 += cells_per_pass) {
        const uint64_t cell = cell0 + gtid / (uint64_t)lanes;
        int ones = 0;
        if (cell < ncell) {
            const uint4 *cp = bits16 + cell * (uint64_t)vecs_per_cell;
            for (int v = sub; v < vecs_per_cell; v += lanes) {
                const uint4 q = __ldg(cp + v);
                ones += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
            }
        }
        for (int d = lanes >> 1; d > 0; d >>= 1) ones += __shfl_xor_sync(0xFFFFFFFFu, ones, d);
        if (sub == 0 && cell < ncell) zc[cell] = g - ones;
    }
}

// Cells narrower than 16 bytes (g = 8 .. 64): one lane per cell, byte loads.
__global__ void __launch_bounds__(256) k_zero_counts_small(const uint8_t *__restrict__ bits,
                                                           int32_t *__restrict__ zc, uint64_t ncell,
                                                           int bytes_per_cell, int g)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t cell = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; cell < ncell; cell += stride) {
        int ones = 0;
        for (int b = 0; b < bytes_per_cell; b++) ones += __popc((uint32_t)bits[cell * bytes_per_cell + b]);
        zc[cell] = g - ones;
    }
}

// Scalars of the read-out:
//   flow count  = mean_i( -C ln(ZR(i)/C) ), ZR == 0 -> evaluate at 1, flag saturated
//                 (pkg/src/dhsa/estimator.py:26-34, dhla.py:121-128)
//   psi         = 1 - exp(-flow / C)                          (dhla.py:130-134)
//   denom       = g (1 - psi^r)                               (dhla.py:184)
// and the "any hot set empty -> no candidates" rule (dhla.py:208-209).
// Sharing-corrected estimate (pkg/src/dhsa/dhla.py:183-189):
//   SZ == 0 -> saturated, evaluate at 1;  SZ >= denom -> 0.0;  else -g ln(SZ/denom).
__device__ __forceinline__ double corrected_estimate(int g, int sz_clamped, double denom)
{
    if ((double)sz_clamped >= denom) return 0.0;
    return -(double)g * log((double)sz_clamped / denom);
}

// The threshold filter `estimate >= theta` (dhla.py:190-194) as an integer cut on the clamped
// SZ: the estimate is non-increasing in SZ, so the passing values are a prefix [1, sz_cut] of
// [1, g] (0 = nothing passes).  Found by a search here so the chain stays on the device; the
// host re-derives the cut with its own libm from the same zero totals when it collects the
// read-out (dhsa_cabi.cu: host_scalars) and re-filters in the -- never yet observed -- case that
// the two disagree, so the decision is the host formula's, not this libm's.
// Called by one full warp: a 32-ary search (two rounds at g = 1024) instead of a bisection --
// every probe is a dependent fp64 log, and the read-out chain is latency-bound.
__device__ __forceinline__ int report_cut(int g, double denom, double theta, uint32_t lane)
{
    int lo = 0, hi = g;  // the answer lies in [lo, hi]; lo = 0 means "nothing passes"
    while (hi > lo) {
        const int step = (hi - lo + 31) / 32;
        int x = lo + ((int)lane + 1) * step;
        if (x > hi) x = hi;
        const unsigned pass = __ballot_sync(0xFFFFFFFFu, corrected_estimate(g, x, denom) >= theta);
        const int cnt = pass == 0xFFFFFFFFu ? 32 : __ffs(~pass) - 1;  // probes are ascending: the passing ones are a prefix
        if (cnt == 32) {
            lo = hi;  // lane 31 probed hi itself
        } else {
            const int fail_at = lo + (cnt + 1) * step < hi ? lo + (cnt + 1) * step : hi;
            lo = lo + cnt * step;
            hi = fail_at - 1;
        }
    }
    return lo;
}

// Called by warp 0 of the CTA that finishes k_hot_sets last.
__device__ __forceinline__ void plan_readout(Control *ctl, int r, int k, int g, double theta, uint32_t lane)
{
    const double cap = (double)g * (double)(1ull << k);
    // per-array terms in parallel (r <= 64: two per lane), summed in array order by lane 0
    double term[2] = {0.0, 0.0};
    int sat = 0, empty = 0;
    for (int h = 0; h < 2; h++) {
        const int i = (int)lane + 32 * h;
        if (i < r) {
            long long z = ctl->zero_totals[i];
            if (z == 0) {
                sat = 1;
                z = 1;
            }
            term[h] = -cap * log((double)z / cap);
            if (ctl->hot_counts[i] == 0) empty = 1;
        }
    }
    sat = __any_sync(0xFFFFFFFFu, sat);
    empty = __any_sync(0xFFFFFFFFu, empty);
    double acc = 0.0;
    for (int i = 0; i < r; i++) acc += __shfl_sync(0xFFFFFFFFu, term[i >> 5], i & 31);
    const double flow = acc / r;
    const double psi = 1.0 - exp(-flow / cap);
    const double denom = g * (1.0 - pow(psi, (double)r));
    const int cut = report_cut(g, denom, theta, lane);
    ctl->stage_counts[lane] = 0;
    ctl->stage_counts[lane + 32] = 0;
    if (lane == 0) {
        ctl->flow_count = flow;
        ctl->flow_saturated = sat;
        ctl->psi = psi;
        ctl->denom = denom;
        ctl->sz_cut = cut;
        ctl->any_empty = empty;
        ctl->n_candidates = 0;
        ctl->n_reports = 0;
        ctl->fail_stage = 0;
        ctl->fail_count = 0;
        ctl->sorted = 0;
    }
}

// Dhla.hot_sets (pkg/src/dhsa/dhla.py:111-119): HE(i) = { j : zc[i][j] < zmin },
// ascending -- as the integer compare zc <= zc_cut, zc_cut = the largest integer below zmin,
// derived on the host from the reference's own float64 formula (dhla.py:45-47); plus the 2^k-bit hot bitmap of each array and ZR(i) = sum_j zc[i][j]
// (dhla.py:126).  One 1024-thread CTA per array; each thread owns 16 consecutive
// cells (64 contiguous bytes of zero counts), so the default 2^14-cell array is
// one pass: thread-local 16-bit hot mask, one block scan, in-order list writes.
// The last CTA to finish computes the scalars above (no extra launch).
#define DHSA_HOT_CPT 16
__global__ void __launch_bounds__(1024) k_hot_sets(const int32_t *__restrict__ zc, int zc_cut, double theta, int r, int k, int g,
                                                   uint32_t *__restrict__ lists,
                                                   uint32_t *__restrict__ bitmaps,
                                                   uint64_t bitmap_words_per_array, Control *ctl)
{
    __shared__ uint32_t warp_count[32];
    __shared__ unsigned long long warp_sum[32];
    __shared__ uint32_t chunk_total_s;
    __shared__ unsigned long long chunk_sum_s;
    __shared__ bool is_last_s;
    const int arr = blockIdx.x;
    const uint64_t m = 1ull << k;
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const int32_t *row = zc + (uint64_t)arr * m;
    uint32_t *list = lists + (uint64_t)arr * m;
    uint32_t *bmp = bitmaps + (uint64_t)arr * bitmap_words_per_array;
    unsigned long long base = 0, total = 0;
    for (uint64_t c0 = 0; c0 < m; c0 += 1024ull * DHSA_HOT_CPT) {
        const uint64_t j0 = c0 + (uint64_t)threadIdx.x * DHSA_HOT_CPT;
        uint32_t hot = 0;
        unsigned long long zs = 0;
        if (j0 + DHSA_HOT_CPT <= m) {
            const int4 *v = reinterpret_cast<const int4 *>(row + j0);
#pragma unroll
            for (int q = 0; q < DHSA_HOT_CPT / 4; q++) {
                const int4 z = v[q];
                hot |= (uint32_t)(z.x <= zc_cut) << (4 * q + 0);
                hot |= (uint32_t)(z.y <= zc_cut) << (4 * q + 1);
                hot |= (uint32_t)(z.z <= zc_cut) << (4 * q + 2);
                hot |= (uint32_t)(z.w <= zc_cut) << (4 * q + 3);
                zs += (unsigned long long)z.x + (unsigned long long)z.y + (unsigned long long)z.z +
                      (unsigned long long)z.w;
            }
        } else {
            for (int q = 0; q < DHSA_HOT_CPT; q++)
                if (j0 + q < m) {
                    const int32_t z = row[j0 + q];
                    hot |= (uint32_t)(z <= zc_cut) << q;
                    zs += (unsigned long long)z;
                }
        }
        // bitmap: two threads share a 32-bit word
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, hot, 1);
        if ((threadIdx.x & 1u) == 0 && j0 < m) bmp[j0 >> 5] = hot | (other << 16);
        // ordered compaction: exclusive scan of the per-thread counts
        const uint32_t cnt = __popc(hot);
        uint32_t inc = cnt;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= (uint32_t)d) inc += t;
        }
        for (int d = 16; d > 0; d >>= 1) zs += __shfl_xor_sync(0xFFFFFFFFu, zs, d);
        if (lane == 31) warp_count[wid] = inc;
        if (lane == 0) warp_sum[wid] = zs;
        __syncthreads();
        if (wid == 0) {
            const uint32_t wc = warp_count[lane];
            uint32_t winc = wc;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, winc, d);
                if (lane >= (uint32_t)d) winc += t;
            }
            unsigned long long ws = warp_sum[lane];
            for (int d = 16; d > 0; d >>= 1) ws += __shfl_xor_sync(0xFFFFFFFFu, ws, d);
            __syncwarp();
            warp_count[lane] = winc - wc;  // exclusive offset of each warp
            if (lane == 31) chunk_total_s = winc;
            if (lane == 0) chunk_sum_s = ws;
        }
        __syncthreads();
        uint32_t pos = (uint32_t)base + warp_count[wid] + (inc - cnt);
        for (uint32_t hbits = hot; hbits; hbits &= hbits - 1) list[pos++] = (uint32_t)(j0 + (__ffs(hbits) - 1));
        base += chunk_total_s;
        total += chunk_sum_s;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctl->hot_counts[arr] = base;
        ctl->zero_totals[arr] = (long long)total;
        __threadfence();
        is_last_s = atomicAdd(&ctl->blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last_s && threadIdx.x < 32) {
        __threadfence();
        plan_readout(ctl, r, k, g, theta, threadIdx.x);
        if (threadIdx.x == 0) ctl->blocks_done = 0;
    }
}

// ------------------------------------------------------------ K3: restore --
//
// Dhla._candidate_hosts (pkg/src/dhsa/dhla.py:198-217).  The reference crosses
// whole hot sets and keeps tuples whose neighbouring blocks agree on their
// k - alpha overlapping bits.  Here the overlap rule is used constructively: a
// partial key fixes the low k - alpha bits of the next block, so only its top
// alpha bits are free -- 2^alpha candidate cells, each tested against the next
// array's hot bitmap.  When the next hot set is smaller than 2^alpha its list is
// walked instead (the reference's own enumeration).  Either way the survivor set
// of every stage is exactly the reference's, so the per-stage counts and the
// CapacityError they trigger (dhla.py:269-273, 294-298) are identical.

__device__ __forceinline__ bool bitmap_test(const uint32_t *bmp, uint32_t idx)
{
    return (bmp[idx >> 5] >> (idx & 31u)) & 1u;
}

// Two bounds travel through the stage kernels.  max_candidates is the reference's bound: a stage
// that produces more partial keys raises CapacityError (dhla.py:269-273, 294-298).  buf_cap
// (<= max_candidates) is what the workspaces hold right now: the library sizes them for the
// default bound and grows them when a stage needs more (dhsa_cabi.cu: restore_collect), so a huge
// "unlimited" max_candidates does not allocate 64 bytes per entry up front.  Every stage counts
// all its survivors either way, so the counts -- and the error they trigger -- are exact.
__device__ __forceinline__ bool stage_blocked(const Control *ctl, int stage_index,
                                              unsigned long long buf_cap)
{
    // stage_index = number of stages already run.  Blocked when some hot set is
    // empty, or an earlier stage overflowed the buffers (then nothing after it runs:
    // either the reference would have raised there, or the host grows the buffers and reruns).
    if (ctl->any_empty) return true;
    for (int s = 0; s < stage_index; s++)
        if (ctl->stage_counts[s] > buf_cap) return true;
    return false;
}

// Stage 1 (_stage_first, pkg/src/dhsa/dhla.py:252-274): (cl0, cl1) in HE0 x HE1,
// b1 = cl0 ^ cl1 is the key's low block; cl2 = cl0 ^ b2 with
// b2 & omask == b1 >> alpha; sub = b1 | (b2 >> (k - alpha)) << k.
__device__ __forceinline__ void stage_first_body(const uint32_t *__restrict__ lists,
                                                 const uint32_t *__restrict__ bitmaps,
                                                 uint64_t bitmap_words_per_array, const DevParams &p,
                                                 unsigned long long buf_cap, uint64_t *__restrict__ out_sub,
                                                 uint32_t *__restrict__ out_cl0, Control *ctl, uint64_t tid,
                                                 uint64_t stride)
{
    if (stage_blocked(ctl, 0, buf_cap)) return;
    const uint64_t m = 1ull << p.k;
    const uint64_t n0 = ctl->hot_counts[0], n1 = ctl->hot_counts[1], n2 = ctl->hot_counts[2];
    const uint64_t next = 1ull << p.alpha;
    const bool by_list = n2 < next;
    const uint64_t E = by_list ? n2 : next;
    const uint64_t total = n0 * n1 * E;
    const int top = p.k - p.alpha;
    const uint32_t omask = (uint32_t)((1ull << top) - 1);
    const uint32_t *he0 = lists, *he1 = lists + m, *he2 = lists + 2 * m;
    const uint32_t *bmp2 = bitmaps + 2 * bitmap_words_per_array;
    for (uint64_t f = tid; f < total; f += stride) {
        const uint64_t t = f % E, pair = f / E;
        const uint32_t cl0 = he0[pair / n1];
        const uint32_t b1 = cl0 ^ he1[pair % n1];
        uint32_t b2;
        bool ok;
        if (by_list) {
            b2 = cl0 ^ he2[t];
            ok = (b1 >> p.alpha) == (b2 & omask);
        } else {
            b2 = ((uint32_t)t << top) | (b1 >> p.alpha);
            ok = bitmap_test(bmp2, cl0 ^ b2);
        }
        if (ok) {
            const unsigned long long pos = atomicAdd(&ctl->stage_counts[0], 1ull);
            if (pos < buf_cap) {
                out_sub[pos] = (uint64_t)b1 | ((uint64_t)(b2 >> top) << p.k);
                out_cl0[pos] = cl0;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_stage_first(const uint32_t *__restrict__ lists,
                                                     const uint32_t *__restrict__ bitmaps,
                                                     uint64_t bitmap_words_per_array, DevParams p,
                                                     unsigned long long buf_cap,
                                                     uint64_t *__restrict__ out_sub,
                                                     uint32_t *__restrict__ out_cl0, Control *ctl)
{
    stage_first_body(lists, bitmaps, bitmap_words_per_array, p, buf_cap, out_sub, out_cl0, ctl,
                     (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

// Stage for array i >= 3 (_stage_next, pkg/src/dhsa/dhla.py:277-299):
// blk = cl0 ^ cl_i must satisfy blk & omask == sub >> (i-1) alpha;
// sub |= (blk >> (k - alpha)) << (k + (i-2) alpha).
__device__ __forceinline__ void stage_next_body(int i, const uint32_t *__restrict__ lists,
                                                const uint32_t *__restrict__ bitmaps,
                                                uint64_t bitmap_words_per_array, const DevParams &p,
                                                unsigned long long buf_cap, const uint64_t *__restrict__ in_sub,
                                                const uint32_t *__restrict__ in_cl0, uint64_t *__restrict__ out_sub,
                                                uint32_t *__restrict__ out_cl0, Control *ctl, uint64_t tid,
                                                uint64_t stride)
{
    const int s = i - 2;  // stages already run
    if (stage_blocked(ctl, s, buf_cap)) return;
    const uint64_t m = 1ull << p.k;
    const uint64_t np = ctl->stage_counts[s - 1], ni = ctl->hot_counts[i];
    const uint64_t next = 1ull << p.alpha;
    const bool by_list = ni < next;
    const uint64_t E = by_list ? ni : next;
    const uint64_t total = np * E;
    const int top = p.k - p.alpha;
    const uint32_t omask = (uint32_t)((1ull << top) - 1);
    const int sh_chk = (i - 1) * p.alpha, sh_put = p.k + (i - 2) * p.alpha;
    const uint32_t *he = lists + (uint64_t)i * m;
    const uint32_t *bmp = bitmaps + (uint64_t)i * bitmap_words_per_array;
    for (uint64_t f = tid; f < total; f += stride) {
        const uint64_t t = f % E, q = f / E;
        const uint64_t sp = in_sub[q];
        const uint32_t cl0 = in_cl0[q];
        const uint32_t want = (uint32_t)(sp >> sh_chk);  // k - alpha bits
        uint32_t blk;
        bool ok;
        if (by_list) {
            blk = cl0 ^ he[t];
            ok = want == (blk & omask);
        } else {
            blk = ((uint32_t)t << top) | want;
            ok = bitmap_test(bmp, cl0 ^ blk);
        }
        if (ok) {
            const unsigned long long pos = atomicAdd(&ctl->stage_counts[s], 1ull);
            if (pos < buf_cap) {
                out_sub[pos] = sp | ((uint64_t)(blk >> top) << sh_put);
                out_cl0[pos] = cl0;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_stage_next(int i, const uint32_t *__restrict__ lists,
                                                    const uint32_t *__restrict__ bitmaps,
                                                    uint64_t bitmap_words_per_array, DevParams p,
                                                    unsigned long long buf_cap,
                                                    const uint64_t *__restrict__ in_sub,
                                                    const uint32_t *__restrict__ in_cl0,
                                                    uint64_t *__restrict__ out_sub,
                                                    uint32_t *__restrict__ out_cl0, Control *ctl)
{
    stage_next_body(i, lists, bitmaps, bitmap_words_per_array, p, buf_cap, in_sub, in_cl0, out_sub, out_cl0, ctl,
                    (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

// Tail of _candidate_hosts (pkg/src/dhsa/dhla.py:213-216): drop partials with bits
// above key_width, keep those whose dh0 reproduces cl0.  A key determines cl0 and
// the tuple <-> (sub, cl0) map is one-to-one, so survivors are already distinct.
// The first stage whose survivor count exceeds max_candidates: the numbers of the CapacityError
// text (stage 1, then i - 1 for array i; dhla.py:269-273, 294-298).  A stage that only overflowed
// the buffers (<= max_candidates) stops the scan: later counts are not final until the rerun.
__device__ __forceinline__ void record_capacity_failure(Control *ctl, int n_stages, unsigned long long buf_cap,
                                                        unsigned long long max_candidates)
{
    if (ctl->any_empty) return;
    for (int st = 0; st < n_stages; st++) {
        if (ctl->stage_counts[st] > max_candidates) {
            ctl->fail_stage = st + 1;
            ctl->fail_count = ctl->stage_counts[st];
            return;
        }
        if (ctl->stage_counts[st] > buf_cap) return;
    }
}

__global__ void __launch_bounds__(256) k_verify_keys(int n_stages, DevParams p, unsigned long long buf_cap,
                                                     unsigned long long max_candidates,
                                                     const uint64_t *__restrict__ in_sub,
                                                     const uint32_t *__restrict__ in_cl0,
                                                     uint64_t *__restrict__ keys, Control *ctl)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) record_capacity_failure(ctl, n_stages, buf_cap, max_candidates);
    if (stage_blocked(ctl, n_stages, buf_cap)) return;
    const uint64_t np = ctl->stage_counts[n_stages - 1];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < np; q += stride) {
        const uint64_t sub = in_sub[q];
        if (sub >> p.key_width) continue;
        if (dh0_of(p, sub) != in_cl0[q]) continue;
        const unsigned long long pos = atomicAdd(&ctl->n_candidates, 1ull);
        keys[pos] = sub;  // pos < np <= buf_cap
    }
}

// ------------------------------- K4: re-estimate + threshold filter + order --

// Multi-GPU, partitioned read-out: after the OR reduce-scatter the merged copy of byte range q of the
// sketch lives on rank q only (multi.py merge_partitioned).  A kernel that needs a candidate's cells
// reads each from its owner, over NVLink through the peer-mapped sketch pointers, instead of every
// rank first copying the whole merged sketch.  Cuts fall on cell boundaries.
#define DHSA_MAX_OWNERS 16
struct CellOwners {
    const uint8_t *base[DHSA_MAX_OWNERS];  // start of owner q's sketch (this rank's own bits for q = rank)
    uint64_t cut[DHSA_MAX_OWNERS + 1];     // owner q holds bytes [cut[q], cut[q + 1])
    int n;
};

template <bool OWNED>
__device__ __forceinline__ const uint8_t *cell_bytes(const uint8_t *__restrict__ bits, const CellOwners &own, uint64_t off)
{
    if (!OWNED) return bits + off;
    int q = 0;
    while (q + 1 < own.n && off >= own.cut[q + 1]) q++;
    return own.base[q] + off;
}

template <bool OWNED>
__device__ __forceinline__ uint4 ld_cell_v4(const uint8_t *ptr)
{
    if (!OWNED) return *reinterpret_cast<const uint4 *>(ptr);
    uint4 x;  // possibly peer memory: past L1, like k_or_merge
    asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(ptr));
    return x;
}

template <bool OWNED>
__device__ __forceinline__ uint32_t ld_cell_u8(const uint8_t *ptr)
{
    if (!OWNED) return *ptr;
    uint32_t x;
    asm volatile("ld.global.cv.u8 %0, [%1];" : "=r"(x) : "l"(ptr));
    return x;
}

// SZ of one key: g - popcount(AND of its r cells) (pkg/src/dhsa/dhla.py:136-143).
// One warp per key, 16-byte vectors when cells are at least 16 bytes wide.
template <bool OWNED>
__device__ __forceinline__ int shared_zero_count_warp(const uint8_t *__restrict__ bits, const CellOwners &own,
                                                      const DevParams &p, uint64_t key, uint32_t lane)
{
    const uint32_t d0 = dh0_of(p, key);
    const uint64_t g = 1ull << p.log2g, bpe = g >> 3;
    int ones = 0;
    if (bpe >= 16) {
        const int vecs = (int)(bpe >> 4);
        for (int v = lane; v < vecs; v += 32) {
            uint4 acc = make_uint4(~0u, ~0u, ~0u, ~0u);
            for (int i = 0; i < p.r; i++) {
                const uint64_t cell = ((uint64_t)i << p.k) | index_of(p, key, d0, i);
                const uint4 q = ld_cell_v4<OWNED>(cell_bytes<OWNED>(bits, own, cell * bpe) + (uint64_t)v * 16);
                acc.x &= q.x, acc.y &= q.y, acc.z &= q.z, acc.w &= q.w;
            }
            ones += __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        }
    } else {
        for (int b = lane; b < (int)bpe; b += 32) {
            uint32_t acc = 0xFFu;
            for (int i = 0; i < p.r; i++) {
                const uint64_t cell = ((uint64_t)i << p.k) | index_of(p, key, d0, i);
                acc &= ld_cell_u8<OWNED>(cell_bytes<OWNED>(bits, own, cell * bpe) + b);
            }
            ones += __popc(acc);
        }
    }
    for (int d = 16; d > 0; d >>= 1) ones += __shfl_xor_sync(0xFFFFFFFFu, ones, d);
    return (int)g - ones;
}

template <bool OWNED>
__device__ __forceinline__ void shared_zero_counts_body(const uint8_t *__restrict__ bits, const CellOwners &own,
                                                        const DevParams &p, const uint64_t *__restrict__ keys, uint64_t n,
                                                        int32_t *__restrict__ sz)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nwarps) {
        const int z = shared_zero_count_warp<OWNED>(bits, own, p, keys[t], lane);
        if (lane == 0) sz[t] = z;
    }
}

__global__ void __launch_bounds__(256) k_shared_zero_counts(const uint8_t *__restrict__ bits, DevParams p,
                                                            const uint64_t *__restrict__ keys, uint64_t n,
                                                            int32_t *__restrict__ sz)
{
    shared_zero_counts_body<false>(bits, CellOwners(), p, keys, n, sz);
}

__global__ void __launch_bounds__(256) k_shared_zero_counts_owned(CellOwners own, DevParams p,
                                                                  const uint64_t *__restrict__ keys, uint64_t n,
                                                                  int32_t *__restrict__ sz)
{
    shared_zero_counts_body<true>(nullptr, own, p, keys, n, sz);
}

// Sort key of one report.  The reference orders by (-estimate, host)
// (dhla.py:195); the estimate is strictly decreasing in the clamped SZ below
// denom and 0.0 from denom on, so (class, host) with class = clamped SZ, or one
// shared value for the zero class, sorts identically with integers only.
//   bits 63..33 class | bits 32..1 host | bit 0 saturated
#define DHSA_ZERO_CLASS 0x7FFFFFFFull
__device__ __forceinline__ uint64_t pack_report(int sz, double denom, uint64_t host)
{
    const int szc = sz == 0 ? 1 : sz;
    const uint64_t cls = ((double)szc >= denom) ? DHSA_ZERO_CLASS : (uint64_t)szc;
    return (cls << 33) | (host << 1) | (uint64_t)(sz == 0);
}

// Verify + re-estimate in one launch: one warp per partial key of the last stage -- key-width
// cut, dh0(key) == cl0 (dhla.py:213-216; k_verify_keys is the stand-alone form behind
// _candidate_hosts), then SZ and the threshold filter (dhla.py:183-194) as the integer compare
// max(SZ, 1) <= ctl->sz_cut.  Every verified key is kept with its SZ (keys[], cand_sz[]) so the
// filter can be re-applied with another cut without touching the bits again (k_refilter).
template <bool OWNED>
__device__ __forceinline__ void verify_reestimate_body(int n_stages, const DevParams &p, unsigned long long buf_cap,
                                                       const uint64_t *__restrict__ in_sub,
                                                       const uint32_t *__restrict__ in_cl0,
                                                       const uint8_t *__restrict__ bits, const CellOwners &own,
                                                       uint64_t *__restrict__ keys,
                                                       int32_t *__restrict__ cand_sz, uint64_t *__restrict__ packed,
                                                       Control *ctl, uint64_t warp, uint64_t nwarps)
{
    if (stage_blocked(ctl, n_stages, buf_cap)) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t np = ctl->stage_counts[n_stages - 1];
    const double denom = ctl->denom;
    const int cut = ctl->sz_cut;
    for (uint64_t q = warp; q < np; q += nwarps) {
        const uint64_t sub = in_sub[q];
        if (sub >> p.key_width) continue;           // warp-uniform
        if (dh0_of(p, sub) != in_cl0[q]) continue;  // warp-uniform
        const int sz = shared_zero_count_warp<OWNED>(bits, own, p, sub, lane);
        if (lane == 0) {
            const unsigned long long pos = atomicAdd(&ctl->n_candidates, 1ull);  // < np <= buf_cap
            keys[pos] = sub;
            cand_sz[pos] = sz;
            if ((sz == 0 ? 1 : sz) <= cut) packed[atomicAdd(&ctl->n_reports, 1ull)] = pack_report(sz, denom, sub);
        }
    }
}

__global__ void __launch_bounds__(256) k_verify_reestimate(int n_stages, DevParams p, unsigned long long buf_cap,
                                                           unsigned long long max_candidates,
                                                           const uint64_t *__restrict__ in_sub,
                                                           const uint32_t *__restrict__ in_cl0,
                                                           const uint8_t *__restrict__ bits,
                                                           uint64_t *__restrict__ keys, int32_t *__restrict__ cand_sz,
                                                           uint64_t *__restrict__ packed, Control *ctl)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) record_capacity_failure(ctl, n_stages, buf_cap, max_candidates);
    verify_reestimate_body<false>(n_stages, p, buf_cap, in_sub, in_cl0, bits, CellOwners(), keys, cand_sz, packed, ctl,
                                  ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                                  ((uint64_t)gridDim.x * blockDim.x) >> 5);
}

// the same with every candidate cell read from the rank that owns its merged copy
__global__ void __launch_bounds__(256) k_verify_reestimate_owned(int n_stages, DevParams p, unsigned long long buf_cap,
                                                                 unsigned long long max_candidates,
                                                                 const uint64_t *__restrict__ in_sub,
                                                                 const uint32_t *__restrict__ in_cl0, CellOwners own,
                                                                 uint64_t *__restrict__ keys, int32_t *__restrict__ cand_sz,
                                                                 uint64_t *__restrict__ packed, Control *ctl)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) record_capacity_failure(ctl, n_stages, buf_cap, max_candidates);
    verify_reestimate_body<true>(n_stages, p, buf_cap, in_sub, in_cl0, nullptr, own, keys, cand_sz, packed, ctl,
                                 ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                                 ((uint64_t)gridDim.x * blockDim.x) >> 5);
}

// The filter again, over the verified keys and their SZ, with a cut handed in by the host
// (n_reports was zeroed by the caller).
__global__ void __launch_bounds__(256) k_refilter(const uint64_t *__restrict__ keys, const int32_t *__restrict__ cand_sz,
                                                  int cut, uint64_t *__restrict__ packed, Control *ctl)
{
    const uint64_t n = ctl->n_candidates;
    const double denom = ctl->denom;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const int sz = cand_sz[t];
        if ((sz == 0 ? 1 : sz) <= cut) packed[atomicAdd(&ctl->n_reports, 1ull)] = pack_report(sz, denom, keys[t]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->sz_cut = cut;
}

struct ReportOut {
    uint64_t host;
    double estimate;
    int32_t saturated;
    int32_t shared_zero_count;
};

// One packed report -> the row handed back to the caller (SuperPointReport, dhla.py:50-54).
__device__ __forceinline__ ReportOut unpack_report(uint64_t w, int g, double denom)
{
    const uint64_t cls = w >> 33;
    const int sat = (int)(w & 1ull);
    ReportOut r;
    r.host = (w >> 1) & 0xFFFFFFFFull;
    r.saturated = sat;
    if (cls == DHSA_ZERO_CLASS) {
        r.estimate = 0.0;
        r.shared_zero_count = -1;  // not recoverable from the zero class; unused by callers
    } else {
        r.estimate = corrected_estimate(g, (int)cls, denom);
        r.shared_zero_count = sat ? 0 : (int)cls;
    }
    return r;
}

// Only for report lists too long for the single-CTA sorter, which emits its own rows.
__global__ void __launch_bounds__(256) k_emit_reports(const uint64_t *__restrict__ packed, int g,
                                                      ReportOut *__restrict__ out, const Control *ctl)
{
    const uint64_t n = ctl->n_reports;
    const double denom = ctl->denom;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride)
        out[t] = unpack_report(packed[t], g, denom);
}

// ------------------------------------------------------------------- sort --
// Ascending sort of u64 words.  Up to SORT_SMEM_MAX entries one CTA sorts in
// shared memory with the count read from the device (no host round trip);
// beyond that the host drives the global bitonic passes below.
#define DHSA_SORT_SMEM_MAX 8192

// emit != nullptr: the sorted words are packed reports and their rows are written too
// (sort + emit in one launch; the read-out chain is latency-bound, every launch is ~5 us).
// emit != nullptr: the sorted words are packed reports and their rows are written too
// (sort + emit in one launch; the read-out chain is latency-bound, every launch is ~5 us).
// As the chain's last kernel it also gathers what the host reads back into ONE block behind the
// control block -- the window counters and the first DHSA_HEAD_ROWS report rows -- so a read-out
// costs one device-to-host copy, not three.
#define DHSA_HEAD_ROWS 256
struct Readback {
    Control c;
    ReportOut head[DHSA_HEAD_ROWS];
};

__global__ void __launch_bounds__(1024) k_sort_small(uint64_t *__restrict__ data,
                                                     const unsigned long long *__restrict__ n_ptr,
                                                     Control *ctl, ReportOut *__restrict__ emit, int g,
                                                     const unsigned long long *__restrict__ counters,
                                                     ReportOut *__restrict__ head)
{
    extern __shared__ uint64_t sm[];
    const uint64_t n = *n_ptr;
    if (counters && threadIdx.x < 4) ctl->counters[threadIdx.x] = counters[threadIdx.x];
    if (n > DHSA_SORT_SMEM_MAX) return;
    uint32_t len = 1;
    while (len < n) len <<= 1;
    for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) sm[t] = t < n ? data[t] : ~0ull;
    __syncthreads();
    for (uint32_t kk = 2; kk <= len; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) {
                const uint32_t x = t ^ j;
                if (x > t) {
                    const uint64_t a = sm[t], b = sm[x];
                    const bool up = (t & kk) == 0;
                    if ((a > b) == up) {
                        sm[t] = b;
                        sm[x] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) data[t] = sm[t];
    if (emit) {
        const double denom = ctl->denom;
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
            const ReportOut row = unpack_report(sm[t], g, denom);
            emit[t] = row;
            if (head && t < DHSA_HEAD_ROWS) head[t] = row;
        }
    }
    if (threadIdx.x == 0 && ctl) ctl->sorted = 1;
}

__global__ void __launch_bounds__(256) k_sort_pad(uint64_t *__restrict__ data, uint64_t n, uint64_t len)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = n + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len; t += stride) data[t] = ~0ull;
}

__global__ void __launch_bounds__(256) k_bitonic_pass(uint64_t *__restrict__ data, uint64_t len, uint64_t kk,
                                                      uint64_t j)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len; t += stride) {
        const uint64_t x = t ^ j;
        if (x > t) {
            const uint64_t a = data[t], b = data[x];
            const bool up = (t & kk) == 0;
            if ((a > b) == up) {
                data[t] = b;
                data[x] = a;
            }
        }
    }
}

// ------------------------------------------------------------- K5: merge --
//
// dhsa.dhla.merge (pkg/src/dhsa/dhla.py:305-318) is a bitwise OR of two bit
// arrays.  Multi-GPU: each rank owns a byte range of the sketch and ORs that
// range of every peer's private sketch into its own copy, reading the peers
// straight over NVLink (peer / IPC-mapped pointers) with 16-byte loads -- a
// reduce-scatter whose reduction is OR, which NCCL does not offer.
#define DHSA_MAX_PEERS 16
struct PeerPtrs {
    const uint4 *p[DHSA_MAX_PEERS];
};

__global__ void __launch_bounds__(256) k_or_merge(uint4 *__restrict__ dst, PeerPtrs peers, int n_peers,
                                                  uint64_t vec_lo, uint64_t vec_hi)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = vec_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vec_hi; v += stride) {
        uint4 acc = dst[v];
        for (int q = 0; q < n_peers; q++) {
            uint4 x;
            // peer memory: bypass L1 so a later merge never sees a stale line
            asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                         : "l"(peers.p[q] + v));
            acc.x |= x.x, acc.y |= x.y, acc.z |= x.z, acc.w |= x.w;
        }
        dst[v] = acc;
    }
}

__global__ void __launch_bounds__(256) k_copy_slice(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                                    uint64_t vec_lo, uint64_t vec_hi)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = vec_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vec_hi; v += stride) {
        uint4 x;
        asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                     : "l"(src + v));
        dst[v] = x;
    }
}

// all-gather of the per-range zero counts (int32 per cell) from a peer's counts region
__global__ void __launch_bounds__(256) k_copy_words(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src,
                                                    uint64_t lo, uint64_t hi)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < hi; w += stride) {
        uint32_t x;
        asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(x) : "l"(src + w));
        dst[w] = x;
    }
}

// ------------------------------------------------- exact oracle on the GPU --
// exact_oracle (pkg/src/dhsa/ingest.py:159-176): the exact number of distinct opposites of
// every candidate host, the ground truth FPR / FNR are scored against.  The reference sorts
// and uniques 64-bit (cand << 32 | opp) keys with numpy; at 10^8..10^9 packets that is minutes.
// Here: an open-addressing hash set of whole pairs (linear probing, 64-bit atomicCAS); the
// lane that wins a pair's insertion bumps its candidate's counter in a second open-addressing
// table keyed by the candidate.  Both tables store key + 1 so that 0 means empty (pair
// 0xFFFFFFFF'FFFFFFFF and host 0xFFFFFFFF are tracked in two dedicated slots of the header).
struct ExactTables {
    unsigned long long *pairs;  // pair_cap slots
    unsigned long long pair_mask;
    unsigned long long *hosts;  // host_cap slots: (host + 1) << 32 | count
    unsigned long long host_mask;
    unsigned long long *header;  // [0] distinct pairs, [1] distinct hosts, [2] overflow flag,
                                 // [3] all-ones pair seen, [4] count of host 0xFFFFFFFF
};

#define DHSA_EXACT_MAX_PROBES 2048ull

__device__ __forceinline__ void exact_bump_host(const ExactTables &t, uint32_t host)
{
    if (host == 0xFFFFFFFFu) {
        if (atomicAdd(t.header + 4, 1ull) == 0ull) atomicAdd(t.header + 1, 1ull);
        return;
    }
    const unsigned long long tag = ((unsigned long long)host + 1ull) << 32;
    unsigned long long slot = mix64((unsigned long long)host) & t.host_mask;
    for (unsigned long long probes = 0; probes <= t.host_mask && probes < DHSA_EXACT_MAX_PROBES;
         probes++, slot = (slot + 1) & t.host_mask) {
        unsigned long long cur = t.hosts[slot];
        if (cur == 0ull) {
            const unsigned long long prev = atomicCAS(t.hosts + slot, 0ull, tag | 1ull);
            if (prev == 0ull) {
                atomicAdd(t.header + 1, 1ull);
                return;
            }
            cur = prev;
        }
        if ((cur >> 32) == (tag >> 32)) {
            atomicAdd(t.hosts + slot, 1ull);  // count lives in the low 32 bits (< 2^32 distinct opposites)
            return;
        }
    }
    atomicExch(t.header + 2, 1ull);  // table full
}

template <typename SRC>
__global__ void __launch_bounds__(256) k_exact_insert(SRC src, ExactTables t)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nvec = src.vectors();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t pol = policy_evict_first();
    uint32_t on_time = 0, late = 0;
    for (uint64_t base = warp0 * 32; base < nvec; base += nwarps * 32) {
        const uint64_t v = base + lane;
        typename SRC::Raw raw;
        src.load(raw, v, pol);
        uint32_t cs[4], os[4];
        bool ok[4];
        src.unpack(raw, v, cs, os, ok, on_time, late);
        if (*reinterpret_cast<volatile unsigned long long *>(t.header + 2)) break;  // flagged full: the result is void anyway
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (!ok[j]) continue;
            const unsigned long long key = ((unsigned long long)cs[j] << 32) | (unsigned long long)os[j];
            if (key == ~0ull) {
                if (atomicExch(t.header + 3, 1ull) == 0ull) {
                    atomicAdd(t.header + 0, 1ull);
                    exact_bump_host(t, cs[j]);
                }
                continue;
            }
            const unsigned long long stored = key + 1ull;
            unsigned long long slot = mix64(key) & t.pair_mask;
            bool placed = false;
            // A table under its planned load never probes far; a long probe run means it is (nearly) full:
            // flag it and stop -- walking a full table from every lane would be quadratic -- the caller rebuilds larger.
            for (unsigned long long probes = 0; probes <= t.pair_mask && probes < DHSA_EXACT_MAX_PROBES;
                 probes++, slot = (slot + 1) & t.pair_mask) {
                unsigned long long cur = t.pairs[slot];
                if (cur == 0ull) {
                    cur = atomicCAS(t.pairs + slot, 0ull, stored);
                    if (cur == 0ull) {  // this lane inserted the pair: one more distinct opposite of cs[j]
                        atomicAdd(t.header + 0, 1ull);
                        exact_bump_host(t, cs[j]);
                        placed = true;
                        break;
                    }
                }
                if (cur == stored) {
                    placed = true;
                    break;
                }
            }
            if (!placed) atomicExch(t.header + 2, 1ull);
        }
    }
}

// Hosts with at least min_count distinct opposites -> (host, count) rows, unordered.
__global__ void __launch_bounds__(256) k_exact_collect(ExactTables t, unsigned long long min_count,
                                                       unsigned long long *__restrict__ out, unsigned long long cap,
                                                       unsigned long long *__restrict__ n_out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t slot = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; slot <= t.host_mask; slot += stride) {
        const unsigned long long cur = t.hosts[slot];
        if (cur == 0ull) continue;
        const unsigned long long count = cur & 0xFFFFFFFFull, host = (cur >> 32) - 1ull;
        if (count >= min_count) {
            const unsigned long long pos = atomicAdd(n_out, 1ull);
            if (pos < cap) out[pos] = (host << 32) | count;  // sorts by host
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && t.header[4] >= min_count && t.header[4] > 0) {
        const unsigned long long pos = atomicAdd(n_out, 1ull);
        if (pos < cap) out[pos] = (0xFFFFFFFFull << 32) | (t.header[4] & 0xFFFFFFFFull);
    }
}

// ---------------------------------------------- synthetic trace generator --
// generate_trace's per-record half (pkg/src/dhsa/ingest.py:128-151) on the device: flows are
// laid out host-major (host h owns flow indices [prefix[h], prefix[h+1]), its destinations a
// ramp from bases[h], so they are distinct by construction, ingest.py:129-133), every flow is
// repeated `dup` times (duplicate_factor, :135-137), the stream is shuffled and time-ordered
// (:143-148).  Output position p takes record perm(p): a 4-round Feistel network over the
// smallest even-width bit field covering M = flows * dup, cycle-walked into [0, M) -- a
// bijection, so each flow appears exactly `dup` times with no sort and no 8 GB permutation
// array; timestamps rise linearly with p (sorted by construction).  Pure integer arithmetic
// on counters: the numpy restatement in oracle/ reproduces every byte.
struct TraceSpec {
    const uint32_t *hosts;        // n_hosts distinct addresses
    const uint64_t *prefix;       // n_hosts + 1 exclusive prefix sums of the cardinalities
    const uint32_t *bases;        // first destination of each host's ramp
    uint32_t n_hosts;
    uint64_t flows;               // prefix[n_hosts]
    uint64_t total;               // flows * dup
    uint64_t perm_key;
    uint32_t half_bits;           // Feistel half width
    uint32_t start_ts, window_seconds;
};

__device__ __forceinline__ uint64_t trace_permute(uint64_t p, const TraceSpec &t)
{
    const uint64_t mask = (1ull << t.half_bits) - 1ull;
    uint64_t x = p;
    do {
        uint64_t l = (x >> t.half_bits) & mask, r = x & mask;
#pragma unroll
        for (int rnd = 0; rnd < 4; rnd++) {
            const uint64_t f = mix64(r ^ ((t.perm_key + (uint64_t)rnd) * 0x9E3779B97F4A7C15ULL)) & mask;
            const uint64_t nl = r;
            r = l ^ f;
            l = nl;
        }
        x = (l << t.half_bits) | r;
    } while (x >= t.total);
    return x;
}

// records_out (12-byte IPPR records) and/or cand_out / opp_out (host-order uint32) for output
// positions [p_lo, p_hi); any of the three outputs may be null.
__global__ void __launch_bounds__(256) k_generate_trace(TraceSpec t, uint64_t p_lo, uint64_t p_hi,
                                                        uint32_t *__restrict__ records_out,
                                                        uint32_t *__restrict__ cand_out,
                                                        uint32_t *__restrict__ opp_out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = p_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p_hi; p += stride) {
        const uint64_t f = trace_permute(p, t) % t.flows;
        uint32_t lo = 0, hi = t.n_hosts;  // largest h with prefix[h] <= f
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (t.prefix[mid] <= f) lo = mid; else hi = mid;
        }
        const uint32_t src = t.hosts[lo];
        const uint32_t dst = t.bases[lo] + (uint32_t)(f - t.prefix[lo]);
        const uint64_t q = p - p_lo;
        if (records_out) {
            // ts = start + floor(p * window / total), exact in 128-bit arithmetic
            const uint64_t hi64 = __umul64hi(p, (uint64_t)t.window_seconds), lo64 = p * (uint64_t)t.window_seconds;
            uint64_t ts;
            if (hi64 == 0) {
                ts = lo64 / t.total;
            } else {  // p * window >= 2^64: split the division (total < 2^63 here)
                const unsigned __int128 num = ((unsigned __int128)hi64 << 64) | lo64;
                ts = (uint64_t)(num / t.total);
            }
            records_out[3 * q + 0] = t.start_ts + (uint32_t)ts;
            records_out[3 * q + 1] = __byte_perm(src, 0, 0x0123);  // network byte order on the wire
            records_out[3 * q + 2] = __byte_perm(dst, 0, 0x0123);
        }
        if (cand_out) cand_out[q] = src;
        if (opp_out) opp_out[q] = dst;
    }
}

// ------------------------------------------- hash group, forward and inverse --
// dhg.forward_many (pkg/src/dhsa/dhg.py:203-210): the r estimator indices of each key.
__global__ void __launch_bounds__(256) k_forward_many(DevParams p, const uint64_t *__restrict__ keys, uint64_t n,
                                                      uint64_t *__restrict__ indices)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint64_t a = keys[t];
        const uint32_t d0 = dh0_of(p, a);
        for (int i = 0; i < p.r; i++) indices[t * p.r + i] = index_of(p, a, d0, i);
    }
}

// dhg.reconstruct_key / reconstruct_many (pkg/src/dhsa/dhg.py:161-185, 213-233): rebuild the key
// of one full r-tuple of indices; accepted iff every pair of neighbouring blocks agrees on its
// k - alpha overlapping bits, no bit lies above key_width and dh0(key) reproduces index 0 -- the
// predicate the stage kernels apply incrementally (k_stage_first / _next / k_verify_keys).
// keys[t] is written either way (the reference returns "garbage where not ok" too, the same
// garbage: the OR of the shifted blocks).
__global__ void __launch_bounds__(256) k_reconstruct_many(DevParams p, const uint64_t *__restrict__ tuples, uint64_t n,
                                                          uint64_t *__restrict__ keys, uint8_t *__restrict__ ok_out)
{
    const int top = p.k - p.alpha;
    const uint64_t omask = (1ull << top) - 1ull;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint64_t *tp = tuples + t * p.r;
        const uint64_t cl0 = tp[0];
        uint64_t blk = cl0 ^ tp[1];
        uint64_t key = blk;
        bool ok = true;
        for (int i = 2; i < p.r; i++) {
            const uint64_t nxt = cl0 ^ tp[i];
            ok = ok && (blk >> p.alpha) == (nxt & omask);
            key |= (nxt >> top) << (p.k + (i - 2) * p.alpha);
            blk = nxt;
        }
        ok = ok && (key >> p.key_width) == 0;
        ok = ok && (mix64(p.state_dh0 ^ key) & (uint64_t)p.kmask) == cl0;
        keys[t] = key;
        ok_out[t] = ok ? 1 : 0;
    }
}

// ------------------------------------------------------------ L2 probes --
// Random-address 32-bit operations into a buffer that fits L2: the ceiling the
// scan's sketch traffic runs against.  Addresses come from a multiply-xorshift
// of a counter, so consecutive lanes hit unrelated sectors, like hashed cells.
__device__ __forceinline__ uint32_t probe_hash(uint64_t x)
{
    x *= 0x9E3779B97F4A7C15ULL;
    x ^= x >> 29;
    x *= 0xBF58476D1CE4E5B9ULL;
    return (uint32_t)(x >> 32);
}

// KIND 0: RED.OR   1: 32-bit load   2: four loads + one RED per five operations (do the two share a
// limit?)   3: 256-bit load of a whole sector (the flow-cache lookup's shape)
template <int KIND>
__global__ void __launch_bounds__(256) k_probe_l2(uint32_t *__restrict__ words, uint32_t word_mask,
                                                  uint64_t ops, uint32_t *__restrict__ sink)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ops; t += stride * 4) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint64_t q = t + (uint64_t)u * stride;
            if (q < ops) {
                const uint32_t hsh = probe_hash(q);
                uint32_t *wp = words + (hsh & word_mask);
                if (KIND == 0) {
                    red_or(wp, 1u << (hsh >> 27));
                } else if (KIND == 1) {
                    acc += ld_sketch(wp);
                } else if (KIND == 2) {
                    acc += ld_sketch(wp);
                    if (u == 3) red_or(words + (probe_hash(q ^ 0x5555555555ull) & word_mask), 1u << (hsh >> 27));
                } else {
                    unsigned long long e[4];
                    ld_fc_set(reinterpret_cast<const unsigned long long *>(words + (hsh & word_mask & ~7u)), e);
                    acc += (uint32_t)(e[0] ^ e[1] ^ e[2] ^ e[3]);
                }
            }
        }
    }
    if (KIND != 0 && acc == 0x12345678u) *sink = acc;
}

}  // namespace dhsa
