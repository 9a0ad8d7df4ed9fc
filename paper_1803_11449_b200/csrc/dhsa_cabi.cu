// dhsa_cabi.cu -- host side of libdhsa_b200.so: the C ABI declared in
// include/dhsa_b200.h over the sm_100a kernels in dhsa_device.cuh.
//
// One dhsa_sketch owns: the bit array in HBM, a launch stream, the device
// control block of the read-out chain with its pinned host mirror, and lazily
// grown workspaces (zero counts, hot lists/bitmaps, ping-pong partial-key
// buffers, packed reports).  No CPU implementation of any step lives here: if
// CUDA is unavailable every call fails with a negative code.
#include "../../include/dhsa_b200.h"
#include "dhsa_device.cuh"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

using namespace dhsa;


// ------------------------------------------------------------------ errors --

static thread_local char g_err[512];

static int fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

static int cuda_fail(cudaError_t e, const char *what)
{
    return fail(-(1000 + (int)e), "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CU(expr)                                          \
    do {                                                  \
        cudaError_t e_ = (expr);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
    } while (0)

#define NEED(ptr)                                                        \
    do {                                                                 \
        if (!(ptr)) return fail(DHSA_ECONFIG, "null argument: %s", #ptr); \
    } while (0)

// ------------------------------------------------------------------ handle --

#ifndef DHSA_COPY_NT_DEFAULT
#define DHSA_COPY_NT_DEFAULT true
#endif
#ifndef DHSA_READOUT_CTAS_PER_SM
#define DHSA_READOUT_CTAS_PER_SM 4   // grid of the stage / verify / re-estimate kernels (grid-stride loops)
#endif
static const uint64_t kCounterBytes = 256;   // device counters kept behind the bit array
static const uint64_t kPinnedReports = DHSA_HEAD_ROWS;  // report rows that come back with the control block
static const uint32_t kPinnedBoundaries = 64;  // report rows copied back inside the read-out graph
static const int kStageBufs = 3;            // staging buffers of the host-input pipeline
static const uint64_t kStagePackets = 1ull << 22;  // packets per staged chunk (16 MiB per array)
static const int kHostSlots = 6;                    // pinned accumulation slots for host input
static const uint64_t kHostSlotPackets = 1ull << 20;  // packets per slot (4 MiB per array)

// Host batches are appended into pinned slots and a slot is copied to the device and scanned once
// it is full (or at the next barrier / read-out): the reference engine hands over 65,536-pair
// batches (pkg/src/dhsa/engine.py:22,78-86), and one H2D copy + one kernel launch per batch is
// launch-latency-bound at ~1 Gpps.  Callers on several threads reserve disjoint ranges of a slot
// under a short lock and fill them in parallel outside it.
struct HostSlot {
    uint32_t *cand, *opp;  // pinned
    cudaEvent_t dma_done;  // the last copy out of this slot has finished
    bool dma_pending;      // ... and was queued: wait for it before refilling
    int state;             // 0 free, 1 open (accepting reservations), 2 closed (writers may still be copying)
    bool submitting;       // a thread holding the sketch lock is queueing this slot
    uint64_t reserved;     // packets handed out to writers
    uint64_t copied;       // packets whose memcpy has finished
};

struct dhsa_sketch {
    dhsa_params_t params;
    DevParams dp;
    int device;
    int sm_count;
    int scan_mode;
    int last_mode_used;     // kernel variant of the last vectorised scan launch (what auto resolved to)
    uint64_t nbytes;        // exact payload, r * 2^k * g/8
    uint64_t alloc_bytes;   // padded to 16 B
    uint8_t *bits;
    cudaStream_t own_stream, stream;
    cudaStream_t copy_stream;
    std::mutex mu;
    uint64_t launches;
    cudaEvent_t bridge_ev;  // orders a foreign producer stream with the launch stream (dhsa_update_device_from)
    int occ[5][2];          // resident CTAs per SM of the scan kernel of [mode][packet source] (0 = not asked yet)
    bool fc_opted_in[2];    // the flow-cache kernel's >48 KB dynamic shared memory was granted on this device
    bool fc_gated_opted_in[2];  // ... and its gated instantiation's (device-gated auto launches)
    uint64_t mutation_seq;  // bumped by every call that can change the bits

    // flow cache of scan mode 3
    unsigned long long *fcache;
    unsigned long long *fc_stats;  // device: flow-cache lookups, hits
    uint32_t fc_sets;              // requested size in sets; the table is allocated on first use
    bool fc_dirty;                 // holds entries since the last clear
    unsigned long long *fc_stats_host;  // pinned snapshot of fc_stats for the auto policy
    cudaEvent_t fc_stats_ev;
    cudaStream_t stat_stream;      // the snapshots travel on their own stream: off the launch stream's critical path
    cudaEvent_t fc_scan_ev;        // launch stream -> stat_stream: the scan whose counters the snapshot wants is done
    bool fc_stats_pending;
    bool auto_fell_back;           // auto mode: this window's flows do not repeat, use the 5-access kernel
    bool auto_cache_trusted;       // auto mode: the last counters seen (this window's or an earlier one's) showed repeats

    // read-out workspaces
    Readback *rb, *rb_host;  // control block + window counters + first report rows: device, and its pinned mirror
    Control *ctl;           // = &rb->c
    Control *ctl_host;      // = &rb_host->c
    int32_t *zc;            // ncell; lives behind the bit array and the window counters, inside the same allocation, so
                            // a peer that has the sketch mapped can read this rank's zero counts too
    bool zc_given;          // s->zc holds counts handed in by the caller for the next read-out call
    CellOwners owners;      // n > 0: partitioned read-out -- zero counts as gathered into s->zc, cells from their owners
    uint64_t owners_seq;    // bumped whenever the owner table changes (it is baked into the read-out graph)
    uint32_t *lists;        // r * 2^k
    uint32_t *bitmaps;      // r * bitmap_words
    uint64_t bitmap_words;  // per array
    uint64_t cand_cap;      // entries in the buffers below
    uint64_t *sub[2];
    uint32_t *cl0[2];
    uint64_t *keys;         // verified keys, then sorted candidates
    int32_t *cand_sz;       // SZ of each verified key (k_verify_reestimate), kept for k_refilter
    uint64_t *packed;       // packed reports (padded to a power of two for the big sorter)
    uint64_t packed_cap;
    ReportOut *reports;
    uint64_t *hosts_in;     // shared_zero_counts input
    int32_t *sz_out;
    uint64_t hosts_in_cap;
    void *host_tmp;         // pinned scratch of the array-returning read-out calls (grown on demand)
    uint64_t host_tmp_bytes;

    // the read-out chain as a CUDA graph (captured once per theta / max_candidates / workspace)
    cudaGraphExec_t restore_graph;
    double graph_theta;
    uint64_t graph_max_candidates;
    uint64_t graph_cand_cap;
    uint64_t graph_owners_seq;
    uint64_t graph_kernels;
    bool graph_disabled;
    ReportOut *reports_pinned;      // the first kPinnedReports rows land here with the control block
    cudaEvent_t restore_ev;         // read-out enqueued by dhsa_restore_begin has landed in the pinned mirrors
    unsigned long long *tally_pinned;  // the 4 window counters (record tally, flow-cache lookups / hits) as of the last read-out
    bool restore_pending;
    uint64_t restore_max_candidates;
    double restore_theta;
    uint64_t restore_seq;           // mutation_seq when the pending read-out was queued

    // record streams
    unsigned long long *tally;      // device: records fed, records dropped
    uint32_t *plan_block_max;
    long long *plan_carry;
    PlanBoundary *plan_out;
    uint32_t *plan_rise;            // blocks in which the running window maximum rises
    uint8_t *plan_pinned;           // count (8 bytes) + the first kPinnedBoundaries boundaries
    unsigned int *plan_count;
    uint64_t plan_blocks_cap;
    uint32_t plan_out_cap;

    // host-input staging
    uint32_t *stage_cand[kStageBufs], *stage_opp[kStageBufs];
    cudaEvent_t ev_copied[kStageBufs], ev_scanned[kStageBufs];
    bool staging_ready;
    uint64_t stage_seq;

    // host input: pinned accumulation slots filled by the calling threads (in parallel, outside mu)
    HostSlot hslots[kHostSlots];
    bool hslots_ready;
    unsigned hcur;            // slot taking reservations
    std::mutex hmu;           // lock order: mu before hmu; never wait for mu while holding hmu
    std::condition_variable hcv;
};

// ---- per-device cache of the expensive-to-create pieces of a sketch ---------------------------
// The reference creates one Dhla per window (pkg/src/dhsa/engine.py:63).  Page-locking 48 MB of
// host memory, allocating the device staging ring and the flow-cache table cost tens of
// milliseconds -- more than scanning a 100M-packet window -- so a destroyed sketch hands them to
// the next one created on the same device instead of freeing them (at most kCachedSets of each).
struct HostRingRes {
    uint32_t *cand[kHostSlots], *opp[kHostSlots];
    cudaEvent_t dma_done[kHostSlots];
};
struct StagingRes {
    uint32_t *cand[kStageBufs], *opp[kStageBufs];
    cudaEvent_t copied[kStageBufs], scanned[kStageBufs];
};
struct FlowCacheRes {
    unsigned long long *table;
    uint32_t sets;
};
static const size_t kCachedSets = 2;
struct DeviceCache {
    std::mutex mu;
    std::vector<HostRingRes> rings;
    std::vector<StagingRes> stagings;
    std::vector<FlowCacheRes> tables;
};
static DeviceCache g_cache[64];
static DeviceCache *cache_of(int device) { return device >= 0 && device < 64 ? &g_cache[device] : nullptr; }

static const unsigned long long kPolicyMinSample = DHSA_POLICY_MIN_SAMPLE;  // packets before the auto policy trusts a counter
static const uint64_t kGatedLaunchMin = 8 * DHSA_GATE_SAMPLE;  // one launch at least this long is sampled and gated on the device
static void consume_policy_snapshots(dhsa_sketch *s, bool window_ends);
static int flush_host_locked(dhsa_sketch *s);

static int use_device(const dhsa_sketch *s)
{
    CU(cudaSetDevice(s->device));
    return DHSA_OK;
}

static int grid_for(const dhsa_sketch *s, uint64_t work_items, int block, int max_blocks_per_sm)
{
    uint64_t want = (work_items + (uint64_t)block - 1) / (uint64_t)block;
    uint64_t cap = (uint64_t)s->sm_count * (uint64_t)max_blocks_per_sm;
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

static int ilog2_exact(int64_t v)
{
    int l = 0;
    while ((1ll << l) < v) l++;
    return l;
}

// The DhgParams rules (pkg/src/dhsa/dhg.py:78-105), re-checked at the boundary.
static int validate(const dhsa_params_t *p)
{
    if (p->r < 3) return fail(DHSA_ECONFIG, "r must satisfy r >= 3 (got r=%d)", p->r);
    if (p->r > 64) return fail(DHSA_ECONFIG, "r must satisfy r <= 64 (got r=%d)", p->r);
    if (p->g < 8 || (p->g & (p->g - 1)))
        return fail(DHSA_ECONFIG, "g must be a power of two >= 8 for byte-packed estimators (got g=%d)", p->g);
    if (p->g > (1 << 30)) return fail(DHSA_ECONFIG, "g must satisfy g <= 2^30 (got g=%d)", p->g);
    if (p->k < 1 || p->k > 30) return fail(DHSA_ECONFIG, "k must satisfy 1 <= k <= 30 (got k=%d)", p->k);
    if (p->key_width < 8 || p->key_width > 32)
        return fail(DHSA_ECONFIG, "key_width must satisfy 8 <= key_width <= 32 (got %d)", p->key_width);
    if (p->k > p->key_width)
        return fail(DHSA_ECONFIG, "k must satisfy k <= key_width (got k=%d, key_width=%d)", p->k, p->key_width);
    if (p->alpha < 1 || p->alpha > p->k)
        return fail(DHSA_ECONFIG, "alpha must satisfy 1 <= alpha <= k (got alpha=%d, k=%d)", p->alpha, p->k);
    const int cover = (p->r - 2) * p->alpha + p->k;
    if (cover < p->key_width)
        return fail(DHSA_ECONFIG, "block coverage must satisfy (r-2)*alpha + k >= key_width (got (%d-2)*%d+%d=%d < %d)",
                    p->r, p->alpha, p->k, cover, p->key_width);
    if (cover > 64)
        return fail(DHSA_ECONFIG, "partial keys are staged in 64-bit words: (r-2)*alpha + k <= 64 (got %d)", cover);
    return DHSA_OK;
}

extern "C" int dhsa_abi_version(void) { return DHSA_ABI_VERSION; }
extern "C" const char *dhsa_last_error(void) { return g_err; }

static uint64_t zero_counts_bytes(const dhsa_sketch *s) { return (s->dp.ncell * sizeof(int32_t) + 15) & ~15ull; }

static void free_workspaces(dhsa_sketch *s)
{
    cudaFree(s->lists);
    cudaFree(s->bitmaps);
    for (int b = 0; b < 2; b++) {
        cudaFree(s->sub[b]);
        cudaFree(s->cl0[b]);
    }
    cudaFree(s->keys);
    cudaFree(s->cand_sz);
    cudaFree(s->packed);
    cudaFree(s->reports);
    cudaFree(s->hosts_in);
    cudaFree(s->sz_out);
    s->lists = nullptr, s->bitmaps = nullptr, s->keys = nullptr, s->packed = nullptr, s->cand_sz = nullptr;
    s->reports = nullptr, s->hosts_in = nullptr, s->sz_out = nullptr;
    s->sub[0] = s->sub[1] = nullptr, s->cl0[0] = s->cl0[1] = nullptr;
    s->cand_cap = s->packed_cap = s->hosts_in_cap = 0;
}

static int create_locked(dhsa_sketch *s, const dhsa_params_t *params, int device)
{
    s->params = *params;
    s->device = device;
    CU(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device));
    s->scan_mode = DHSA_SCAN_AUTO;
    s->fc_sets = 1u << 20;
    const uint64_t m = 1ull << params->k;
    s->nbytes = (uint64_t)params->r * m * ((uint64_t)params->g / 8);
    s->alloc_bytes = (s->nbytes + 15) & ~15ull;
    DevParams &d = s->dp;
    d.r = params->r, d.k = params->k, d.alpha = params->alpha, d.key_width = params->key_width;
    d.log2g = ilog2_exact(params->g);
    d.kmask = (uint32_t)(m - 1);
    d.gmask = (uint32_t)(params->g - 1);
    d.state_dh0 = params->state_dh0, d.state_h1 = params->state_h1;
    d.ncell = (uint64_t)params->r * m;
    d.nwords = s->alloc_bytes / 4;
    s->bitmap_words = m >= 32 ? m / 32 : 1;
    // the window's counters (record tally, flow-cache statistics) sit right behind the
    // bit array, so a window reset is ONE memset
    // [bits | window counters | zero counts]: one allocation, one CUDA IPC handle for everything a peer reads
    CU(cudaMalloc(&s->bits, s->alloc_bytes + kCounterBytes + zero_counts_bytes(s)));
    s->zc = reinterpret_cast<int32_t *>(s->bits + s->alloc_bytes + kCounterBytes);
    CU(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    s->stream = s->own_stream;
    CU(cudaMalloc(&s->rb, sizeof(Readback)));
    s->ctl = &s->rb->c;
    s->tally = reinterpret_cast<unsigned long long *>(s->bits + s->alloc_bytes);
    s->fc_stats = s->tally + 2;
    CU(cudaMallocHost(&s->rb_host, sizeof(Readback)));
    memset(s->rb_host, 0, sizeof(Readback));
    s->ctl_host = &s->rb_host->c;
    s->reports_pinned = s->rb_host->head;
    s->tally_pinned = s->rb_host->c.counters;
    CU(cudaEventCreateWithFlags(&s->restore_ev, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&s->bridge_ev, cudaEventDisableTiming));
    s->graph_disabled = getenv("DHSA_NO_GRAPH") != nullptr;
    CU(cudaMemsetAsync(s->bits, 0, s->alloc_bytes + kCounterBytes, s->stream));
    CU(cudaMemsetAsync(s->rb, 0, sizeof(Readback), s->stream));
    CU(cudaStreamSynchronize(s->stream));
    CU(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            DHSA_SORT_SMEM_MAX * (int)sizeof(uint64_t)));
    return DHSA_OK;
}

// ---- parked sketches --------------------------------------------------------------------------
// The reference builds a new Dhla for every window and drops it after the restore
// (pkg/src/dhsa/engine.py:63,165-176).  On the device that is the expensive way round: creating a
// sketch, its first read-out (64 MB of stage workspaces, the captured read-out graph) and freeing
// it all again cost 40-80 ms -- several times the scan of a 100M-packet window.  So dhsa_destroy
// parks up to kParkedPerKey sketches per (device, parameters) and kParkedTotal overall, zeroed and back in their initial
// state, and dhsa_create hands a parked one out again.  dhsa_release_cached() frees them.
static const size_t kParkedPerKey = 2;
static const size_t kParkedTotal = 6;
static std::mutex g_parked_mu;
static std::vector<dhsa_sketch *> g_parked;

static int clear_flow_cache_locked(dhsa_sketch *s, bool clear_stats);
static int order_after_snapshot(dhsa_sketch *s);

static bool same_key(const dhsa_sketch *s, const dhsa_params_t *p, int device)
{
    const dhsa_params_t &x = s->params;
    return s->device == device && x.r == p->r && x.g == p->g && x.k == p->k && x.alpha == p->alpha &&
           x.key_width == p->key_width && x.state_dh0 == p->state_dh0 && x.state_h1 == p->state_h1;
}

static int destroy_for_real(dhsa_sketch *s);

// back to the state dhsa_create leaves a sketch in (its stream is drained)
static int scrub_for_parking(dhsa_sketch *s)
{
    std::lock_guard<std::mutex> lk(s->mu);
    if (s->hslots_ready) {  // batches nobody read are dropped with the window they belonged to
        std::lock_guard<std::mutex> hl(s->hmu);
        for (int i = 0; i < kHostSlots; i++) {
            if (s->hslots[i].submitting || (s->hslots[i].state != 0 && s->hslots[i].copied != s->hslots[i].reserved))
                return -1;  // a writer is still inside: not a sketch to recycle
            s->hslots[i].state = 0, s->hslots[i].reserved = s->hslots[i].copied = 0;
        }
    }
    s->stream = s->own_stream;
    s->scan_mode = DHSA_SCAN_AUTO;
    s->fc_sets = 1u << 20;
    s->launches = 0;
    s->restore_pending = false;
    s->zc_given = false;
    s->owners.n = 0;
    s->owners_seq++;
    s->auto_cache_trusted = false;  // the next owner's traffic is not this one's
    if (int rc = order_after_snapshot(s)) return rc;
    CU(cudaMemsetAsync(s->bits, 0, s->alloc_bytes + kCounterBytes, s->stream));
    if (int rc = clear_flow_cache_locked(s, false)) return rc;
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

extern "C" int dhsa_release_cached(void)
{
    std::vector<dhsa_sketch *> victims;
    {
        std::lock_guard<std::mutex> lk(g_parked_mu);
        victims.swap(g_parked);
    }
    for (dhsa_sketch *s : victims) destroy_for_real(s);
    for (int d = 0; d < 64; d++) {
        DeviceCache &dc = g_cache[d];
        std::lock_guard<std::mutex> lk(dc.mu);
        if (dc.rings.empty() && dc.stagings.empty() && dc.tables.empty()) continue;
        cudaSetDevice(d);
        for (auto &r : dc.rings)
            for (int i = 0; i < kHostSlots; i++) cudaFreeHost(r.cand[i]), cudaFreeHost(r.opp[i]), cudaEventDestroy(r.dma_done[i]);
        for (auto &r : dc.stagings)
            for (int b = 0; b < kStageBufs; b++)
                cudaFree(r.cand[b]), cudaFree(r.opp[b]), cudaEventDestroy(r.copied[b]), cudaEventDestroy(r.scanned[b]);
        for (auto &r : dc.tables) cudaFree(r.table);
        dc.rings.clear(), dc.stagings.clear(), dc.tables.clear();
    }
    (void)cudaGetLastError();
    return DHSA_OK;
}

extern "C" int dhsa_create(const dhsa_params_t *params, int device, dhsa_sketch_t **out)
{
    NEED(params);
    NEED(out);
    *out = nullptr;
    int rc = validate(params);
    if (rc) return rc;
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(DHSA_ECONFIG, "device %d out of range (%d visible)", device, ndev);
    CU(cudaSetDevice(device));
    {
        std::lock_guard<std::mutex> lk(g_parked_mu);
        for (size_t i = 0; i < g_parked.size(); i++)
            if (same_key(g_parked[i], params, device)) {
                *out = g_parked[i];
                g_parked.erase(g_parked.begin() + i);
                return DHSA_OK;
            }
    }
    dhsa_sketch *s = new (std::nothrow) dhsa_sketch();  // value-initialised: every pointer null, every flag false
    if (!s) return fail(-1, "out of host memory");
    rc = create_locked(s, params, device);
    if (rc != DHSA_OK) {  // whatever was allocated before the failing call goes back (the message is kept)
        s->device = device;
        destroy_for_real(s);
        return rc;
    }
    *out = s;
    return DHSA_OK;
}

extern "C" int dhsa_destroy(dhsa_sketch_t *s)
{
    if (!s) return DHSA_OK;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
    if (s->stat_stream) cudaStreamSynchronize(s->stat_stream);
    if (getenv("DHSA_NO_SKETCH_CACHE") == nullptr && s->bits && s->own_stream) {
        size_t same = 0;
        {
            std::lock_guard<std::mutex> lk(g_parked_mu);
            for (dhsa_sketch *q : g_parked) same += same_key(q, &s->params, s->device);
        }
        if (same < kParkedPerKey && scrub_for_parking(s) == DHSA_OK) {
            dhsa_sketch *evicted = nullptr;
            {
                std::lock_guard<std::mutex> lk(g_parked_mu);
                if (g_parked.size() >= kParkedTotal) {  // the oldest makes room
                    evicted = g_parked.front();
                    g_parked.erase(g_parked.begin());
                }
                g_parked.push_back(s);
            }
            if (evicted) destroy_for_real(evicted);
            return DHSA_OK;
        }
        (void)cudaGetLastError();
    }
    return destroy_for_real(s);
}

static int destroy_for_real(dhsa_sketch *s)
{
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
    if (s->stat_stream) cudaStreamSynchronize(s->stat_stream);
    free_workspaces(s);
    DeviceCache *dc = cache_of(s->device);
    if (s->staging_ready) {
        StagingRes r;
        for (int b = 0; b < kStageBufs; b++)
            r.cand[b] = s->stage_cand[b], r.opp[b] = s->stage_opp[b], r.copied[b] = s->ev_copied[b], r.scanned[b] = s->ev_scanned[b];
        bool kept = false;
        if (dc) {
            std::lock_guard<std::mutex> lk(dc->mu);
            if (dc->stagings.size() < kCachedSets) dc->stagings.push_back(r), kept = true;
        }
        if (!kept)
            for (int b = 0; b < kStageBufs; b++) {
                cudaFree(r.cand[b]);
                cudaFree(r.opp[b]);
                cudaEventDestroy(r.copied[b]);
                cudaEventDestroy(r.scanned[b]);
            }
    }
    if (s->hslots_ready) {
        HostRingRes r;
        for (int i = 0; i < kHostSlots; i++)
            r.cand[i] = s->hslots[i].cand, r.opp[i] = s->hslots[i].opp, r.dma_done[i] = s->hslots[i].dma_done;
        bool kept = false;
        if (dc) {
            std::lock_guard<std::mutex> lk(dc->mu);
            if (dc->rings.size() < kCachedSets) dc->rings.push_back(r), kept = true;
        }
        if (!kept)
            for (int i = 0; i < kHostSlots; i++) {
                cudaFreeHost(r.cand[i]);
                cudaFreeHost(r.opp[i]);
                cudaEventDestroy(r.dma_done[i]);
            }
    }
    if (s->fcache) {
        bool kept = false;
        if (dc) {
            std::lock_guard<std::mutex> lk(dc->mu);
            if (dc->tables.size() < kCachedSets) dc->tables.push_back(FlowCacheRes{s->fcache, s->dp.fc_sets}), kept = true;
        }
        if (kept) s->fcache = nullptr;
    }
    cudaFree(s->bits);
    cudaFree(s->plan_block_max);
    cudaFree(s->plan_carry);
    cudaFree(s->plan_out);
    cudaFree(s->plan_rise);
    cudaFree(s->plan_count);
    if (s->plan_pinned) cudaFreeHost(s->plan_pinned);
    cudaFree(s->fcache);
    if (s->fc_stats_host) {
        cudaFreeHost(s->fc_stats_host);
        cudaEventDestroy(s->fc_stats_ev);
    }
    cudaFree(s->rb);
    if (s->rb_host) cudaFreeHost(s->rb_host);
    if (s->host_tmp) cudaFreeHost(s->host_tmp);
    if (s->restore_ev) cudaEventDestroy(s->restore_ev);
    if (s->bridge_ev) cudaEventDestroy(s->bridge_ev);
    if (s->restore_graph) cudaGraphExecDestroy(s->restore_graph);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    if (s->stat_stream) {
        cudaStreamDestroy(s->stat_stream);
        cudaEventDestroy(s->fc_scan_ev);
    }
    (void)cudaGetLastError();
    delete s;
    return DHSA_OK;
}

// The flow cache asserts "this key's bits are in the sketch": it must be emptied
// whenever bits can disappear (reset, upload).  Stream-ordered with the scans.
// A counter snapshot still travelling on the side stream must have read the counters before the launch stream zeroes
// them (stream-ordered: nobody waits on the host).
static int order_after_snapshot(dhsa_sketch *s)
{
    if (s->fc_stats_pending && s->stat_stream) CU(cudaStreamWaitEvent(s->stream, s->fc_stats_ev, 0));
    return DHSA_OK;
}

static int clear_flow_cache_locked(dhsa_sketch *s, bool clear_stats)
{
    if (int rc = order_after_snapshot(s)) return rc;
    // a hit-rate snapshot still in flight belongs to the window that ends here: the auto policy must not
    // judge the next window by it (the copy may still land in fc_stats_host; nothing reads it unasked)
    consume_policy_snapshots(s, true);
    s->fc_stats_pending = false;
    s->auto_fell_back = false;  // a new window may repeat flows again
    if (!s->fcache || !s->fc_dirty) return DHSA_OK;
    // entries carry the epoch they were written in: bumping it empties the table without touching it
    const uint32_t epoch_max = (uint32_t)((1ull << (32 - s->dp.fc_tag_bits)) - 1);
    if (s->dp.fc_epoch >= epoch_max) {
        CU(cudaMemsetAsync(s->fcache, 0, (size_t)32 * s->dp.fc_sets, s->stream));
        s->dp.fc_epoch = 1;
    } else {
        s->dp.fc_epoch++;
    }
    if (clear_stats) CU(cudaMemsetAsync(s->fc_stats, 0, 3 * sizeof(unsigned long long), s->stream));
    s->fc_dirty = false;
    return DHSA_OK;
}

// Sets actually allocated for a requested size: the largest power of two not above it, and at
// least 2g sets -- a 32-bit entry holds the 32 - log2(sets) key bits the set index leaves plus
// log2(g) bits of h1(opp), and needs at least one bit for the epoch.
static int flow_cache_log2_sets(const dhsa_sketch *s)
{
    int l = 0;
    while ((2ull << l) <= (uint64_t)s->fc_sets) l++;
    if (l < s->dp.log2g + 1) l = s->dp.log2g + 1;
    return l;
}

static bool flow_cache_supported(const dhsa_sketch *s) { return s->dp.log2g + 1 <= 27; }

static int ensure_flow_cache_locked(dhsa_sketch *s)
{
    const uint32_t sets = 1u << flow_cache_log2_sets(s);
    if (s->fcache && s->dp.fc_sets == sets) return DHSA_OK;
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(s->fcache);
    s->fcache = nullptr;
    if (DeviceCache *dc = cache_of(s->device)) {  // a table a destroyed sketch left behind (cleared below: epoch restart)
        std::lock_guard<std::mutex> lk(dc->mu);
        for (size_t i = 0; i < dc->tables.size(); i++)
            if (dc->tables[i].sets == sets) {
                s->fcache = dc->tables[i].table;
                dc->tables.erase(dc->tables.begin() + i);
                break;
            }
    }
    if (!s->fcache) CU(cudaMalloc(&s->fcache, (size_t)32 * sets));
    s->dp.fc_sets = sets;
    s->dp.fc_shift = 32 - flow_cache_log2_sets(s);
    s->dp.fc_tag_bits = s->dp.fc_shift + s->dp.log2g;  // <= 31: the table has at least 2g sets
    s->dp.fc_epoch = (uint32_t)((1ull << (32 - s->dp.fc_tag_bits)) - 1);  // = epoch_max: the clear below zeroes the table
    s->dp.fcache = s->fcache;
    s->dp.fc_stats = s->fc_stats;
    s->fc_dirty = true;
    return clear_flow_cache_locked(s, true);
}

extern "C" int dhsa_set_flow_cache(dhsa_sketch_t *s, uint64_t n_sets)
{
    NEED(s);
    if (n_sets < 1024 || n_sets > (1ull << 27))  // slot indices are 32-bit with 0xFFFFFFFF reserved: sets * 8 < 2^32
        return fail(DHSA_ECONFIG, "flow cache size must satisfy 1024 <= n_sets <= 2^27 (got %llu)",
                    (unsigned long long)n_sets);
    std::lock_guard<std::mutex> lk(s->mu);
    s->fc_sets = (uint32_t)n_sets;
    return DHSA_OK;
}

extern "C" int dhsa_flow_cache_stats(dhsa_sketch_t *s, uint64_t *lookups, uint64_t *hits)
{
    NEED(s);
    NEED(lookups);
    NEED(hits);
    *lookups = *hits = 0;
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    unsigned long long v[2];
    CU(cudaMemcpyAsync(v, s->fc_stats, sizeof v, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    *lookups = v[0], *hits = v[1];
    return DHSA_OK;
}

extern "C" int dhsa_reset(dhsa_sketch_t *s)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;  // batches handed over before the reset belong to the old window
    s->mutation_seq++;
    if (int rc = order_after_snapshot(s)) return rc;
    CU(cudaMemsetAsync(s->bits, 0, s->alloc_bytes + kCounterBytes, s->stream));  // bits and every counter
    return clear_flow_cache_locked(s, false);
}

extern "C" int dhsa_sketch_bytes(const dhsa_sketch_t *s, uint64_t *nbytes)
{
    NEED(s);
    NEED(nbytes);
    *nbytes = s->nbytes;
    return DHSA_OK;
}

extern "C" int dhsa_bits_device_ptr(dhsa_sketch_t *s, void **bits_dev)
{
    NEED(s);
    NEED(bits_dev);
    *bits_dev = s->bits;
    return DHSA_OK;
}

static int switch_stream_locked(dhsa_sketch *s, cudaStream_t next)
{
    if (next == s->stream) return DHSA_OK;
    // work already queued on the old stream must precede work on the new one
    cudaEvent_t ev;
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CU(cudaEventRecord(ev, s->stream));
    CU(cudaStreamWaitEvent(next, ev, 0));
    CU(cudaEventDestroy(ev));
    s->stream = next;
    return DHSA_OK;
}

extern "C" int dhsa_set_stream(dhsa_sketch_t *s, void *cuda_stream)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    return switch_stream_locked(s, (cudaStream_t)cuda_stream);
}

extern "C" int dhsa_set_own_stream(dhsa_sketch_t *s)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    return switch_stream_locked(s, s->own_stream);
}

extern "C" int dhsa_get_stream(dhsa_sketch_t *s, void **cuda_stream)
{
    NEED(s);
    NEED(cuda_stream);
    *cuda_stream = (void *)s->stream;
    return DHSA_OK;
}

extern "C" int dhsa_set_scan_mode(dhsa_sketch_t *s, int mode)
{
    NEED(s);
    if (mode < 0 || mode > 4) return fail(DHSA_ECONFIG, "scan mode must be 0..4 (got %d)", mode);
    s->scan_mode = mode;
    return DHSA_OK;
}

extern "C" int dhsa_scan_mode_used(const dhsa_sketch_t *s, int *mode)
{
    NEED(s);
    NEED(mode);
    *mode = s->last_mode_used;
    return DHSA_OK;
}

extern "C" int dhsa_launch_count(const dhsa_sketch_t *s, uint64_t *n)
{
    NEED(s);
    NEED(n);
    *n = s->launches;
    return DHSA_OK;
}

// -------------------------------------------------------------------- scan --

template <typename SRC> struct SrcKind;
template <> struct SrcKind<SoaSource> { static const int value = 0; };
template <> struct SrcKind<RecordSource> { static const int value = 1; };

// resident CTAs per SM of `kernel`, asked once per sketch and (mode, packet source)
template <typename K>
static int resident_ctas(dhsa_sketch *s, int mode, int kind, K kernel, int smem, int fallback)
{
    int &occ = s->occ[mode][kind];
    if (!occ && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, smem) != cudaSuccess || occ < 1))
        occ = fallback;
    return occ;
}

template <int R, typename SRC>
static void launch_scan_src(dhsa_sketch *s, int mode, const SRC &src)
{
    uint32_t *w = reinterpret_cast<uint32_t *>(s->bits);
    const uint64_t nvec = src.vectors();
    const int kind = SrcKind<SRC>::value;
    // persistent grid: SMs x resident CTAs of the chosen kernel
#define LAUNCH(KERNEL, FALLBACK_OCC)                                                                       \
    do {                                                                                                   \
        const int occ = resident_ctas(s, mode, kind, KERNEL, 0, FALLBACK_OCC);                             \
        KERNEL<<<grid_for(s, nvec, 256, occ), 256, 0, s->stream>>>(src, w, s->dp);                         \
    } while (0)
    if (s->dp.gate != 0) {
        // the two kernels behind k_auto_decide in a device-gated auto launch: instantiations that first read the
        // verdict, same grids as their plain twins
        if (mode == DHSA_SCAN_TEST_RED) {
            const int occ = resident_ctas(s, mode, kind, k_scan_vec4<R, 1, SRC>, 0, 3);
            k_scan_vec4<R, 1, SRC, true><<<grid_for(s, nvec, 256, occ), 256, 0, s->stream>>>(src, w, s->dp);
        } else {
            auto kernel = k_scan_flowcache<R, SRC, true>;
            const int smem = FcSmem<SRC>::kBytes;
            if (!s->fc_gated_opted_in[kind]) {
                cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                s->fc_gated_opted_in[kind] = true;
            }
            const int occ = resident_ctas(s, DHSA_SCAN_FLOW_CACHE, kind, k_scan_flowcache<R, SRC>, smem, 3);
            kernel<<<grid_for(s, nvec, 256, occ), 256, smem, s->stream>>>(src, w, s->dp);
        }
        s->launches++;
        return;
    }
    switch (mode) {
    case DHSA_SCAN_RED_ONLY: LAUNCH((k_scan_vec4<R, 0, SRC>), 8); break;
    case DHSA_SCAN_TEST_RED: LAUNCH((k_scan_vec4<R, 1, SRC>), 3); break;
    case DHSA_SCAN_TEST_AGG_RED: LAUNCH((k_scan_vec4<R, 2, SRC>), 2); break;
    // flow cache: 4 packets per lane at 3 CTAs/SM measured best on B200 (profiles/r01_flowcache_variants.txt);
    // 8 packets per lane, 4 CTAs/SM (spills) and L2::evict_last table loads were slower or equal; staging the
    // packet stream by TMA was 2-3% faster than register prefetch and is the only form kept
    default: {
        // flow cache: dynamic shared memory (TMA stage rings + miss queues), 3 CTAs per SM.
        // The opt-in to more than 48 KB is per device, hence per sketch.
        auto kernel = k_scan_flowcache<R, SRC>;
        const int smem = FcSmem<SRC>::kBytes;
        if (!s->fc_opted_in[kind]) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            s->fc_opted_in[kind] = true;
        }
        const int occ = resident_ctas(s, DHSA_SCAN_FLOW_CACHE, kind, kernel, smem, 3);
        kernel<<<grid_for(s, nvec, 256, occ), 256, smem, s->stream>>>(src, w, s->dp);
        break;
    }
    }
#undef LAUNCH
    s->launches++;
}

template <typename SRC>
static void launch_scan_any_r(dhsa_sketch *s, int mode, const SRC &src)
{
    switch (s->params.r) {
    case 3: launch_scan_src<3>(s, mode, src); break;
    case 4: launch_scan_src<4>(s, mode, src); break;
    case 5: launch_scan_src<5>(s, mode, src); break;
    default: launch_scan_src<6>(s, mode, src); break;
    }
}

// ---- the auto policy ------------------------------------------------------------------------
// Decided per launch from counters the scan kernels leave behind the bit array, read through
// asynchronous pinned snapshots (never a synchronisation):
//   * flows that do not repeat (after >= 4M lookups, the hit rate PROJECTED for the next stretch of the window is
//     under 0.3, projected_no_repeats): the rest of the WINDOW goes to the 5-access test-first kernel.  Break-even is
//     a hit rate of about 1/3: 1 + 11 (1 - h) requests per packet with the cache against 5 + 5 (1 - h) without.
// (A second rule of an earlier round -- the plain test-first kernel for windows whose candidates are a
// handful of hosts, BASELINE config 4 with the victims as candidates -- was measured again after the
// lookup loop lost its per-slot miss handling: the cache path now scans that window at 205 Gpps
// against 183 for the test-first kernel, so the rule is gone; profiles/r02_config4_ddos_contention.json.)

// Would the flow cache pay over the NEXT stretch of the window, judged from the m lookups and h hits so far?  A cold
// table hides repeats: the first m packets over F equally likely flows find only ~m/2F of their keys.  So the counts
// are projected the way k_auto_decide does it: x = m / F solves (1 - e^-x) / x = (m - h) / m, and the next m packets of
// the same population miss (e^-x - e^-2x) / x of their lookups.  "No repeats" = that projected miss rate above 0.7
// (the break-even of 1 + 11 (1 - hit) requests per packet against 5 + 5 (1 - hit)).
static bool projected_no_repeats(unsigned long long m, unsigned long long h)
{
    if (m == 0) return false;
    const double rho = (double)(m - h) / (double)m;
    double lo = 1e-9, hi = 64.0;
    for (int it = 0; it < 60; it++) {
        const double x = 0.5 * (lo + hi);
        if (-expm1(-x) / x > rho) lo = x; else hi = x;
    }
    const double x = 0.5 * (lo + hi);
    return (exp(-x) - exp(-2.0 * x)) / x > 0.7;
}

static void consume_policy_snapshots(dhsa_sketch *s, bool window_ends)
{
    if (s->fc_stats_pending && cudaEventQuery(s->fc_stats_ev) == cudaSuccess) {
        s->fc_stats_pending = false;
        const unsigned long long lookups = s->fc_stats_host[0], hits = s->fc_stats_host[1], verdict = s->fc_stats_host[2];
        // what the counters say: flows do not repeat (hit rate under 0.3 after enough lookups, or the device's own
        // projection from a gated launch's sample), they do, or nothing yet
        const bool enough = lookups >= kPolicyMinSample;
        const bool no_repeats = verdict == 2 || (verdict == 0 && enough && projected_no_repeats(lookups, hits));
        const bool repeats = verdict == 1 || (enough && !projected_no_repeats(lookups, hits));
        // a snapshot that arrives when its window is over cannot switch the next window's kernel, but it is the prior
        // that decides whether the next long launch is worth gating on the device
        if (no_repeats) s->auto_cache_trusted = false;
        else if (repeats) s->auto_cache_trusted = true;
        if (no_repeats && !window_ends) s->auto_fell_back = true;
    }
    (void)cudaGetLastError();
}

// Which fast kernel this launch uses (lock held).
static int pick_scan_mode_locked(dhsa_sketch *s)
{
    int mode = s->scan_mode;
    if (mode == DHSA_SCAN_AUTO) {
        consume_policy_snapshots(s, false);
        // the fallback is the plain test-first kernel: without repeats there is nothing for warp aggregation to
        // merge either (all-distinct window: 31.6 Gpps against 29.7 with aggregation)
        mode = s->auto_fell_back ? DHSA_SCAN_TEST_RED : DHSA_SCAN_FLOW_CACHE;
    }
    if (mode == DHSA_SCAN_FLOW_CACHE && !flow_cache_supported(s)) mode = DHSA_SCAN_TEST_AGG_RED;
    return mode;
}

static int before_fast_scan_locked(dhsa_sketch *s, int mode)
{
    s->last_mode_used = mode;
    if (mode == DHSA_SCAN_FLOW_CACHE) {
        if (int rc = ensure_flow_cache_locked(s)) return rc;
        s->fc_dirty = true;
    }
    return DHSA_OK;
}

static int after_fast_scan_locked(dhsa_sketch *s, int mode)
{
    if (s->scan_mode == DHSA_SCAN_AUTO && mode == DHSA_SCAN_FLOW_CACHE && !s->fc_stats_pending) {
        if (!s->fc_stats_host) {
            CU(cudaMallocHost(&s->fc_stats_host, 3 * sizeof(unsigned long long)));
            CU(cudaEventCreateWithFlags(&s->fc_stats_ev, cudaEventDisableTiming));
            memset(s->fc_stats_host, 0, 3 * sizeof(unsigned long long));
        }
        if (!s->stat_stream) {
            CU(cudaStreamCreateWithFlags(&s->stat_stream, cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&s->fc_scan_ev, cudaEventDisableTiming));
        }
        // on a side stream behind this scan: a 24-byte copy on the launch stream itself cost every window ~6 us
        // (scan 0.549-0.555 ms in auto mode against 0.542-0.544 with the cache forced).  Whatever zeroes the counters
        // next waits for it (order_after_snapshot), so it never reads a half-cleared block.
        CU(cudaEventRecord(s->fc_scan_ev, s->stream));
        CU(cudaStreamWaitEvent(s->stat_stream, s->fc_scan_ev, 0));
        CU(cudaMemcpyAsync(s->fc_stats_host, s->fc_stats, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           s->stat_stream));
        CU(cudaEventRecord(s->fc_stats_ev, s->stat_stream));
        s->fc_stats_pending = true;
    }
    return DHSA_OK;
}

// The vectorised kernels cover r in 3..6, cells of at least one word, sketches under 16 GiB.
static bool fast_params(const dhsa_sketch *s)
{
    const dhsa_params_t &p = s->params;
    return p.r >= 3 && p.r <= 6 && s->dp.log2g >= 5 && s->dp.nwords <= 0xFFFFFFFFull;
}

// One long launch in auto mode with no evidence yet that flows repeat: the host cannot look at the counters in the
// middle of it, so the device decides (k_auto_decide) -- a sample of DHSA_GATE_SAMPLE packets through the cache, then
// the rest through whichever kernel the sample's projected hit rate calls for.  38 instead of 15 Gpps on an all-distinct
// window; three short extra launches on one that repeats, and only until a window has shown repeats.
static bool wants_gated_launch(const dhsa_sketch *s, int mode, uint64_t packets)
{
    return s->scan_mode == DHSA_SCAN_AUTO && mode == DHSA_SCAN_FLOW_CACHE && !s->auto_cache_trusted &&
           packets >= kGatedLaunchMin;
}

template <typename SRC>
static void launch_scan_gated(dhsa_sketch *s, const SRC &head, const SRC &rest)
{
    launch_scan_any_r(s, DHSA_SCAN_FLOW_CACHE, head);
    k_auto_decide<<<1, 1, 0, s->stream>>>(s->fc_stats, 4 * rest.vectors());
    s->launches++;
    s->dp.gate = 2;
    launch_scan_any_r(s, DHSA_SCAN_TEST_RED, rest);
    s->dp.gate = 1;
    launch_scan_any_r(s, DHSA_SCAN_FLOW_CACHE, rest);
    s->dp.gate = 0;
}

// Launches the scan of n device-resident packets on s->stream (lock held).
static int scan_locked(dhsa_sketch *s, const uint32_t *cand, const uint32_t *opp, uint64_t n)
{
    if (n == 0) return DHSA_OK;
    uint32_t *words = reinterpret_cast<uint32_t *>(s->bits);
    const bool fast = fast_params(s) && (((uintptr_t)cand | (uintptr_t)opp) & 15u) == 0;
    uint64_t done = 0;
    if (fast && n >= 4) {
        const int mode = pick_scan_mode_locked(s);
        if (int rc = before_fast_scan_locked(s, mode)) return rc;
        SoaSource src;
        src.cand4 = reinterpret_cast<const uint4 *>(cand);
        src.opp4 = reinterpret_cast<const uint4 *>(opp);
        src.nvec = n / 4;
        if (wants_gated_launch(s, mode, n)) {
            const uint64_t head = DHSA_GATE_SAMPLE / 4;
            SoaSource rest = src;
            rest.cand4 += head, rest.opp4 += head, rest.nvec -= head;
            src.nvec = head;
            launch_scan_gated(s, src, rest);
            src.nvec += rest.nvec;
        } else {
            launch_scan_any_r(s, mode, src);
        }
        if (int rc = after_fast_scan_locked(s, mode)) return rc;
        done = src.nvec * 4;
    }
    if (done < n) {
        const uint64_t rest = n - done;
        const int grid = grid_for(s, rest, 256, 8);
        if (s->scan_mode == DHSA_SCAN_RED_ONLY)
            k_scan_generic<0><<<grid, 256, 0, s->stream>>>(cand + done, opp + done, rest, words, s->dp);
        else
            k_scan_generic<1><<<grid, 256, 0, s->stream>>>(cand + done, opp + done, rest, words, s->dp);
        s->launches++;
    }
    CU(cudaGetLastError());
    return DHSA_OK;
}

// One orientation of a record segment (lock held): whole quads inside the buffer through the
// fast kernels, ragged ends (and non-fast parameters) through the one-record-per-lane kernel.
static int scan_records_locked(dhsa_sketch *s, const uint8_t *records, uint64_t n_in_buffer, uint64_t rec_lo,
                               uint64_t rec_hi, uint32_t window_seconds, uint32_t window_id, int cand_is_dst,
                               int tally_late)
{
    uint32_t *words = reinterpret_cast<uint32_t *>(s->bits);
    const uint32_t *rec_words = reinterpret_cast<const uint32_t *>(records);
    uint64_t covered_hi = rec_lo;  // records [rec_lo, covered_hi) were handled by the fast kernel
    if (fast_params(s) && ((uintptr_t)records & 15u) == 0) {
        const uint64_t q_lo = rec_lo / 4, q_hi = (rec_hi + 3) / 4, q_buf = n_in_buffer / 4;  // whole quads only
        const uint64_t q_end = q_hi < q_buf ? q_hi : q_buf;
        if (q_end > q_lo) {
            const int mode = pick_scan_mode_locked(s);
            if (int rc = before_fast_scan_locked(s, mode)) return rc;
            RecordSource src;
            src.rec4 = reinterpret_cast<const uint4 *>(records) + 3 * q_lo;
            src.nquads = q_end - q_lo;
            src.first_rec = 4 * q_lo;
            src.rec_lo = rec_lo;
            src.rec_hi = rec_hi;
            src.set_window(window_seconds, window_id);
            src.cand_is_dst = cand_is_dst;
            src.tally = s->tally;
            src.tally_late = tally_late;
            if (wants_gated_launch(s, mode, 4 * src.nquads)) {
                const uint64_t head = DHSA_GATE_SAMPLE / 4;
                RecordSource rest = src;
                rest.rec4 += 3 * head, rest.nquads -= head, rest.first_rec += 4 * head;
                src.nquads = head;
                launch_scan_gated(s, src, rest);
            } else {
                launch_scan_any_r(s, mode, src);
            }
            if (int rc = after_fast_scan_locked(s, mode)) return rc;
            covered_hi = 4 * q_end < rec_hi ? 4 * q_end : rec_hi;
        }
    }
    if (covered_hi < rec_hi) {  // at most 3 trailing records, or everything on the general path
        const int grid = grid_for(s, rec_hi - covered_hi, 256, 8);
        if (s->scan_mode == DHSA_SCAN_RED_ONLY)
            k_scan_records_generic<0><<<grid, 256, 0, s->stream>>>(rec_words, covered_hi, rec_hi, window_seconds,
                                                                   window_id, cand_is_dst, s->tally, tally_late, words, s->dp);
        else
            k_scan_records_generic<1><<<grid, 256, 0, s->stream>>>(rec_words, covered_hi, rec_hi, window_seconds,
                                                                   window_id, cand_is_dst, s->tally, tally_late, words, s->dp);
        s->launches++;
    }
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_update_records_device(dhsa_sketch_t *s, const void *records_dev, uint64_t n_in_buffer,
                                          uint64_t rec_lo, uint64_t rec_hi, uint32_t window_seconds,
                                          uint32_t window_id, int direction)
{
    NEED(s);
    if (rec_lo >= rec_hi) return DHSA_OK;
    NEED(records_dev);
    if (rec_hi > n_in_buffer) return fail(DHSA_EDATA, "record range [%llu, %llu) exceeds the buffer's %llu records",
                                          (unsigned long long)rec_lo, (unsigned long long)rec_hi,
                                          (unsigned long long)n_in_buffer);
    if (window_seconds == 0) return fail(DHSA_ECONFIG, "window_seconds must be positive (got 0)");
    if (direction < 0 || direction > 2) return fail(DHSA_ECONFIG, "direction must be 0 (src), 1 (dst) or 2 (both)");
    if ((uintptr_t)records_dev & 3u) return fail(DHSA_ECONFIG, "record buffer must be 4-byte aligned");
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    s->mutation_seq++;
    const uint8_t *rec = static_cast<const uint8_t *>(records_dev);
    // "both" feeds each record in both orientations (engine.py:191-192): two passes over the segment.
    // Late records are tallied once, by the first pass.
    if (direction == 0 || direction == 2)
        if (int rc = scan_records_locked(s, rec, n_in_buffer, rec_lo, rec_hi, window_seconds, window_id, 0, 1)) return rc;
    if (direction == 1 || direction == 2)
        if (int rc = scan_records_locked(s, rec, n_in_buffer, rec_lo, rec_hi, window_seconds, window_id, 1,
                                         direction == 1)) return rc;
    return DHSA_OK;
}

extern "C" int dhsa_record_tally(dhsa_sketch_t *s, uint64_t *records_fed, uint64_t *records_dropped)
{
    NEED(s);
    NEED(records_fed);
    NEED(records_dropped);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    unsigned long long v[2];
    CU(cudaMemcpyAsync(v, s->tally, sizeof v, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    *records_fed = v[0], *records_dropped = v[1];
    return DHSA_OK;
}

extern "C" int dhsa_record_tally_at_restore(dhsa_sketch_t *s, uint64_t *records_fed, uint64_t *records_dropped)
{
    NEED(s);
    NEED(records_fed);
    NEED(records_dropped);
    std::lock_guard<std::mutex> lk(s->mu);
    if (s->restore_pending) return fail(DHSA_ECONFIG, "the read-out that carries the tally has not been collected");
    *records_fed = s->tally_pinned[0], *records_dropped = s->tally_pinned[1];
    return DHSA_OK;
}

// ---- parallel memcpy for pageable host input ---------------------------------------------
// A pageable cudaMemcpyAsync is a single-threaded copy into the driver's bounce buffer
// (measured 1.4 Gpps = 11 GB/s); PCIe takes 55 GB/s.  So host arrays are copied into pinned
// slots by several host threads -- a small process-wide pool plus the caller -- and DMA'd from
// there.  The reference engine hands over 65,536-pair batches (512 KB), so a job lasts tens of
// microseconds: helpers poll for about 100 us after their last job before they go to sleep, and
// a caller that finds the pool busy with another caller's job simply copies alone.
// Copy into a pinned slot.  The destination is read next by the DMA engine, never by this CPU, so on x86-64 the
// stores can bypass the cache (no read-for-ownership of the destination lines, no eviction of the caller's data):
// 16-byte streaming stores once the destination is aligned.  DHSA_COPY_NT=0 selects plain memcpy.
#if defined(__x86_64__)
#include <emmintrin.h>
static bool copy_nt_enabled()
{
    static const bool on = [] {
        const char *env = getenv("DHSA_COPY_NT");
        return env ? env[0] != '0' : DHSA_COPY_NT_DEFAULT;
    }();
    return on;
}
static void copy_to_pinned(void *dst, const void *src, size_t n)
{
    if (!copy_nt_enabled() || n < 4096) {
        memcpy(dst, src, n);
        return;
    }
    char *d = (char *)dst;
    const char *s = (const char *)src;
    const size_t lead = (16 - ((uintptr_t)d & 15)) & 15;
    if (lead) {
        memcpy(d, s, lead);
        d += lead, s += lead, n -= lead;
    }
    size_t blocks = n / 64;
    for (; blocks; blocks--, d += 64, s += 64) {
        const __m128i a = _mm_loadu_si128((const __m128i *)(s + 0)), b = _mm_loadu_si128((const __m128i *)(s + 16));
        const __m128i c = _mm_loadu_si128((const __m128i *)(s + 32)), e = _mm_loadu_si128((const __m128i *)(s + 48));
        _mm_stream_si128((__m128i *)(d + 0), a);
        _mm_stream_si128((__m128i *)(d + 16), b);
        _mm_stream_si128((__m128i *)(d + 32), c);
        _mm_stream_si128((__m128i *)(d + 48), e);
    }
    _mm_sfence();
    if (n & 63) memcpy(d, s, n & 63);
}
#else
static void copy_to_pinned(void *dst, const void *src, size_t n) { memcpy(dst, src, n); }
#endif

class CopyPool {
public:
    static CopyPool &get()
    {
        static CopyPool *pool = new CopyPool();  // leaked on purpose: no destructor races at exit
        return *pool;
    }
    // dst <- src for both arrays, split into one share per thread (helpers + the caller); returns
    // when every byte is copied.  The two arrays are treated as one run of 2 * bytes_each bytes.
    void copy2(void *d0, const void *s0, void *d1, const void *s1, size_t bytes_each)
    {
        const size_t total = 2 * bytes_each;
        if (n_helpers_ == 0 || total < (128u << 10) || !job_mu_.try_lock()) {
            copy_to_pinned(d0, s0, bytes_each);
            copy_to_pinned(d1, s1, bytes_each);
            return;
        }
        uint32_t shares = n_helpers_ + 1;
        size_t per = ((total + shares - 1) / shares + 4095) & ~(size_t)4095;  // page-sized steps
        if (per < (32u << 10)) per = 32u << 10;
        shares = (uint32_t)((total + per - 1) / per);
        job_ = Job{(char *)d0, (const char *)s0, (char *)d1, (const char *)s1, bytes_each, per, shares};
        done_.store(0, std::memory_order_relaxed);
        const uint64_t gen = gen_.load(std::memory_order_relaxed) + 1;
        gen_.store(gen, std::memory_order_release);  // publishes job_
        if (sleepers_.load(std::memory_order_acquire) > 0) {
            { std::lock_guard<std::mutex> lk(cv_mu_); }
            cv_.notify_all();
        }
        work(gen, shares - 1);  // the caller starts from the last share, helper i from share i
        while (done_.load(std::memory_order_acquire) != shares) cpu_relax();
        job_mu_.unlock();
    }

private:
    static const uint32_t kMaxShares = 65;
    struct Job {
        char *d0;
        const char *s0;
        char *d1;
        const char *s1;
        size_t bytes_each, per;
        uint32_t shares;
    };
    struct alignas(64) Claim {
        std::atomic<uint64_t> gen{0};  // generation of the job this share was last claimed in
    };
    static void cpu_relax()
    {
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#else
        std::this_thread::yield();
#endif
    }
    // Claim shares of job `gen`, starting at `first`: one compare-exchange per share, on its own cache
    // line.  Generations only grow, and a share is claimable only while its mark is OLDER than `gen`:
    // a helper that wakes up late, after its job is over, finds every mark >= its generation and
    // leaves -- so job_ is only ever read by threads the waiting caller still counts.
    void work(uint64_t gen, uint32_t first)
    {
        const uint32_t shares = job_.shares;
        for (uint32_t k = 0; k < shares; k++) {
            const uint32_t i = (first + k) % shares;
            uint64_t seen = claims_[i].gen.load(std::memory_order_acquire);
            if (seen >= gen) {
                if (seen > gen) return;  // a newer job owns the table
                continue;
            }
            if (!claims_[i].gen.compare_exchange_strong(seen, gen, std::memory_order_acq_rel)) {
                if (seen > gen) return;
                continue;
            }
            // Shares beyond the previous job's count can carry marks older than a late helper's own
            // generation: a claim only counts while `gen` is still the current job.  If it is, the job
            // cannot end before this share is done (nobody else can claim it), so job_ is stable below.
            if (gen_.load(std::memory_order_acquire) != gen) return;
            const Job j = job_;
            if (i >= j.shares) continue;
            size_t lo = (size_t)i * j.per, hi = lo + j.per < 2 * j.bytes_each ? lo + j.per : 2 * j.bytes_each;
            if (lo < j.bytes_each) {
                const size_t end = hi < j.bytes_each ? hi : j.bytes_each;
                copy_to_pinned(j.d0 + lo, j.s0 + lo, end - lo);
                lo = end;
            }
            if (hi > lo) copy_to_pinned(j.d1 + (lo - j.bytes_each), j.s1 + (lo - j.bytes_each), hi - lo);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }
    CopyPool()
    {
        // helper threads: DHSA_COPY_THREADS, else up to 6 while leaving two cores to the application
        unsigned hw = std::thread::hardware_concurrency();
        unsigned n = hw > 4 ? (hw - 2 < 6 ? hw - 2 : 6) : (hw > 1 ? hw - 1 : 0);
        if (const char *env = getenv("DHSA_COPY_THREADS")) {
            const long v = strtol(env, nullptr, 10);
            if (v >= 0 && v < (long)kMaxShares) n = (unsigned)v;
        }
        n_helpers_ = n;
        for (unsigned i = 0; i < n; i++) {
            std::thread th([this, i] { run(i); });
            th.detach();
        }
    }
    void run(uint32_t id)
    {
        uint64_t seen = 0;
        auto last = std::chrono::steady_clock::now();
        for (;;) {
            const uint64_t gen = gen_.load(std::memory_order_acquire);
            if (gen != seen) {
                seen = gen;
                work(gen, id);
                last = std::chrono::steady_clock::now();
                continue;
            }
            if (std::chrono::steady_clock::now() - last < std::chrono::microseconds(100)) {
                cpu_relax();
                continue;
            }
            std::unique_lock<std::mutex> lk(cv_mu_);
            sleepers_.fetch_add(1, std::memory_order_acq_rel);
            cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
            sleepers_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    std::mutex job_mu_;  // one job at a time; a caller that finds it taken copies alone
    Job job_{};
    Claim claims_[kMaxShares];
    std::atomic<uint64_t> gen_{0};
    std::atomic<uint32_t> done_{0};
    std::atomic<int> sleepers_{0};
    std::mutex cv_mu_;
    std::condition_variable cv_;
    unsigned n_helpers_ = 0;
};

// Host-only self test of the copy pool (no CUDA call): `threads` callers issue `iterations` two-array copies of
// random sizes up to bytes_each between private buffers at once -- one of them gets the helpers, the others
// copy alone -- and every copy is compared with its source.  The CPU test suite runs it (tests/test_host_logic.py).
extern "C" int dhsa_selftest_copy_pool(uint64_t bytes_each, int iterations, int threads, uint64_t *mismatches)
{
    NEED(mismatches);
    *mismatches = 0;
    if (bytes_each < 64 || iterations < 1 || threads < 1 || threads > 64)
        return fail(DHSA_ECONFIG, "self test needs bytes_each >= 64, iterations >= 1, 1 <= threads <= 64");
    std::atomic<uint64_t> bad{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; t++)
        pool.emplace_back([&, t] {
            std::vector<uint8_t> s0(bytes_each), s1(bytes_each), d0(bytes_each), d1(bytes_each);
            uint64_t x = 0x9E3779B97F4A7C15ull * (uint64_t)(t + 1);
            for (int it = 0; it < iterations; it++) {
                x ^= x << 13, x ^= x >> 7, x ^= x << 17;
                const size_t n = 64 + (size_t)(x % (bytes_each - 63));
                for (size_t i = 0; i < n; i += 61) s0[i] = (uint8_t)(x >> (i & 31)), s1[i] = (uint8_t)(~x >> (i & 15));
                memset(d0.data(), 0xA5, n);
                memset(d1.data(), 0x5A, n);
                CopyPool::get().copy2(d0.data(), s0.data(), d1.data(), s1.data(), n);
                if (memcmp(d0.data(), s0.data(), n) != 0 || memcmp(d1.data(), s1.data(), n) != 0) bad.fetch_add(1);
            }
        });
    for (auto &th : pool) th.join();
    *mismatches = bad.load();
    return DHSA_OK;
}

static bool is_pageable(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// Process-wide pinned bounce ring for pageable record buffers (per device, allocated on first use).
static const int kBounceSlots = 4;
static const uint64_t kBounceBytes = 8ull << 20;
struct BounceRing {
    std::mutex mu;
    bool ready = false;
    uint8_t *buf[kBounceSlots];
    cudaEvent_t done[kBounceSlots];
    bool used[kBounceSlots];
    unsigned next = 0;
};
static BounceRing g_bounce[16];

extern "C" int dhsa_copy_to_device_async(int device, void *dst_dev, const void *src_host, uint64_t nbytes,
                                         void *cuda_stream)
{
    if (nbytes == 0) return DHSA_OK;
    NEED(dst_dev);
    NEED(src_host);
    CU(cudaSetDevice(device));
    cudaStream_t stream = (cudaStream_t)cuda_stream;
    if (!is_pageable(src_host) || device < 0 || device >= 16) {
        CU(cudaMemcpyAsync(dst_dev, src_host, nbytes, cudaMemcpyHostToDevice, stream));
        return DHSA_OK;
    }
    // pageable: several host threads copy into pinned slots, the DMA of a slot overlaps the fill of the next
    BounceRing &r = g_bounce[device];
    std::lock_guard<std::mutex> lk(r.mu);
    if (!r.ready) {
        for (int i = 0; i < kBounceSlots; i++) {
            CU(cudaMallocHost(&r.buf[i], kBounceBytes));
            CU(cudaEventCreateWithFlags(&r.done[i], cudaEventDisableTiming));
            r.used[i] = false;
        }
        r.ready = true;
    }
    for (uint64_t off = 0; off < nbytes; off += kBounceBytes) {
        const uint64_t cnt = nbytes - off < kBounceBytes ? nbytes - off : kBounceBytes;
        const int i = (int)(r.next++ % kBounceSlots);
        if (r.used[i]) CU(cudaEventSynchronize(r.done[i]));
        {   // two halves so the pool's two-array entry point serves a single buffer too
            const uint64_t half = (cnt / 2) & ~63ull;
            if (half) CopyPool::get().copy2(r.buf[i], (const uint8_t *)src_host + off, r.buf[i] + half,
                                            (const uint8_t *)src_host + off + half, half);
            if (cnt > 2 * half) memcpy(r.buf[i] + 2 * half, (const uint8_t *)src_host + off + 2 * half, cnt - 2 * half);
        }
        CU(cudaMemcpyAsync((uint8_t *)dst_dev + off, r.buf[i], cnt, cudaMemcpyHostToDevice, stream));
        CU(cudaEventRecord(r.done[i], stream));
        r.used[i] = true;
    }
    return DHSA_OK;
}

static int cmp_boundary(const void *a, const void *b)
{
    const dhsa_boundary_t *x = static_cast<const dhsa_boundary_t *>(a), *y = static_cast<const dhsa_boundary_t *>(b);
    return (x->position > y->position) - (x->position < y->position);
}

extern "C" int dhsa_plan_windows(dhsa_sketch_t *s, const void *records_dev, uint64_t n_records, uint32_t window_seconds,
                                 int64_t open_window, dhsa_boundary_t *out_host, uint32_t cap, uint32_t *n_out)
{
    NEED(s);
    NEED(n_out);
    *n_out = 0;
    if (n_records == 0) return DHSA_OK;
    NEED(records_dev);
    NEED(out_host);
    if (window_seconds == 0) return fail(DHSA_ECONFIG, "window_seconds must be positive (got 0)");
    if ((uintptr_t)records_dev & 3u) return fail(DHSA_ECONFIG, "record buffer must be 4-byte aligned");
    if (cap == 0) return fail(DHSA_ECONFIG, "boundary capacity must be positive");
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    const uint64_t nblocks = (n_records + DHSA_PLAN_BLOCK - 1) / DHSA_PLAN_BLOCK;
    if (nblocks > 0x7FFFFFFFull) return fail(DHSA_EDATA, "record buffer too large for one plan (%llu records)",
                                             (unsigned long long)n_records);
    if (nblocks > s->plan_blocks_cap || cap > s->plan_out_cap) {
        CU(cudaStreamSynchronize(s->stream));
        const uint64_t nb = nblocks > s->plan_blocks_cap ? nblocks : s->plan_blocks_cap;
        const uint32_t nc = cap > s->plan_out_cap ? cap : s->plan_out_cap;
        cudaFree(s->plan_block_max);
        cudaFree(s->plan_carry);
        cudaFree(s->plan_rise);
        cudaFree(s->plan_out);
        s->plan_block_max = nullptr, s->plan_carry = nullptr, s->plan_out = nullptr, s->plan_rise = nullptr;
        s->plan_blocks_cap = 0, s->plan_out_cap = 0;
        CU(cudaMalloc(&s->plan_block_max, nb * sizeof(uint32_t)));
        CU(cudaMalloc(&s->plan_carry, nb * sizeof(long long)));
        CU(cudaMalloc(&s->plan_rise, nb * sizeof(uint32_t)));
        CU(cudaMalloc(&s->plan_out, (size_t)nc * sizeof(PlanBoundary)));
        if (!s->plan_count) {
            CU(cudaMalloc(&s->plan_count, 2 * sizeof(unsigned int)));  // [0] boundaries, [1] blocks where the maximum rises
            CU(cudaMallocHost(&s->plan_pinned, sizeof(unsigned int) + kPinnedBoundaries * sizeof(PlanBoundary) + 8));
        }
        s->plan_blocks_cap = nb;
        s->plan_out_cap = nc;
    }
    const uint32_t *rec_words = static_cast<const uint32_t *>(records_dev);
    CU(cudaMemsetAsync(s->plan_count, 0, 2 * sizeof(unsigned int), s->stream));
    k_plan_blockmax<<<(unsigned)nblocks, 256, 0, s->stream>>>(rec_words, n_records, window_seconds, s->plan_block_max);
    k_plan_carry<<<1, 1024, 0, s->stream>>>(s->plan_block_max, nblocks, (long long)open_window, s->plan_carry,
                                            s->plan_rise, s->plan_count + 1);
    const unsigned bgrid = (unsigned)(nblocks < 256 ? nblocks : 256);
    k_plan_boundaries<<<bgrid, 256, 0, s->stream>>>(rec_words, n_records, window_seconds, s->plan_carry, s->plan_rise,
                                                    s->plan_count + 1, s->plan_out, cap, s->plan_count);
    s->launches += 3;
    CU(cudaGetLastError());
    // the count and the first few boundaries come back together: one synchronisation per chunk
    unsigned int *n_pinned = reinterpret_cast<unsigned int *>(s->plan_pinned);
    PlanBoundary *b_pinned = reinterpret_cast<PlanBoundary *>(s->plan_pinned + 8);
    const uint32_t first = cap < kPinnedBoundaries ? cap : kPinnedBoundaries;
    CU(cudaMemcpyAsync(n_pinned, s->plan_count, sizeof(unsigned int), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(b_pinned, s->plan_out, (size_t)first * sizeof(PlanBoundary), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    const unsigned int n = *n_pinned;
    if (n > cap) return fail(DHSA_EDATA, "record stream opens %u windows, more than the plan capacity %u", n, cap);
    static_assert(sizeof(PlanBoundary) == sizeof(dhsa_boundary_t), "boundary layouts must match");
    if (n) {
        if (n <= first) {
            memcpy(out_host, b_pinned, (size_t)n * sizeof(PlanBoundary));
        } else {
            CU(cudaMemcpyAsync(out_host, s->plan_out, (size_t)n * sizeof(PlanBoundary), cudaMemcpyDeviceToHost, s->stream));
            CU(cudaStreamSynchronize(s->stream));
        }
        qsort(out_host, n, sizeof(dhsa_boundary_t), cmp_boundary);
    }
    *n_out = n;
    return DHSA_OK;
}

extern "C" int dhsa_update_device(dhsa_sketch_t *s, const uint32_t *cand_dev, const uint32_t *opp_dev, uint64_t n)
{
    NEED(s);
    if (n == 0) return DHSA_OK;
    NEED(cand_dev);
    NEED(opp_dev);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    s->mutation_seq++;
    return scan_locked(s, cand_dev, opp_dev, n);
}

// The same scan for arrays produced on ANOTHER stream (torch's current stream, say): the launch
// stream waits for what that stream has queued so far, and that stream waits for the scan before
// it runs anything queued later -- so the producer may free or overwrite the arrays right after
// the call, and the sketch keeps launching on its own stream.
extern "C" int dhsa_update_device_from(dhsa_sketch_t *s, const uint32_t *cand_dev, const uint32_t *opp_dev, uint64_t n,
                                       void *producer_stream)
{
    NEED(s);
    if (n == 0) return DHSA_OK;
    NEED(cand_dev);
    NEED(opp_dev);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    s->mutation_seq++;
    cudaStream_t ps = (cudaStream_t)producer_stream;
    if (ps == s->stream) return scan_locked(s, cand_dev, opp_dev, n);
    CU(cudaEventRecord(s->bridge_ev, ps));
    CU(cudaStreamWaitEvent(s->stream, s->bridge_ev, 0));
    if (int rc = scan_locked(s, cand_dev, opp_dev, n)) return rc;
    CU(cudaEventRecord(s->bridge_ev, s->stream));
    CU(cudaStreamWaitEvent(ps, s->bridge_ev, 0));
    return DHSA_OK;
}

static int ensure_staging(dhsa_sketch *s)
{
    if (s->staging_ready) return DHSA_OK;
    if (DeviceCache *dc = cache_of(s->device)) {
        std::lock_guard<std::mutex> lk(dc->mu);
        if (!dc->stagings.empty()) {
            const StagingRes r = dc->stagings.back();
            dc->stagings.pop_back();
            for (int b = 0; b < kStageBufs; b++)
                s->stage_cand[b] = r.cand[b], s->stage_opp[b] = r.opp[b], s->ev_copied[b] = r.copied[b], s->ev_scanned[b] = r.scanned[b];
            s->staging_ready = true;
            s->stage_seq = 0;
            return DHSA_OK;
        }
    }
    for (int b = 0; b < kStageBufs; b++) {
        CU(cudaMalloc(&s->stage_cand[b], kStagePackets * 4));
        CU(cudaMalloc(&s->stage_opp[b], kStagePackets * 4));
        CU(cudaEventCreateWithFlags(&s->ev_copied[b], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&s->ev_scanned[b], cudaEventDisableTiming));
    }
    s->staging_ready = true;
    s->stage_seq = 0;
    return DHSA_OK;
}

static int ensure_host_slots(dhsa_sketch *s)
{
    std::lock_guard<std::mutex> lk(s->hmu);
    if (s->hslots_ready) return DHSA_OK;
    HostRingRes cached;
    bool have = false;
    if (DeviceCache *dc = cache_of(s->device)) {
        std::lock_guard<std::mutex> cl(dc->mu);
        if (!dc->rings.empty()) {
            cached = dc->rings.back();
            dc->rings.pop_back();
            have = true;
        }
    }
    for (int i = 0; i < kHostSlots; i++) {
        if (have) {
            s->hslots[i].cand = cached.cand[i], s->hslots[i].opp = cached.opp[i], s->hslots[i].dma_done = cached.dma_done[i];
        } else {
            CU(cudaMallocHost(&s->hslots[i].cand, kHostSlotPackets * 4));
            CU(cudaMallocHost(&s->hslots[i].opp, kHostSlotPackets * 4));
            CU(cudaEventCreateWithFlags(&s->hslots[i].dma_done, cudaEventDisableTiming));
        }
        s->hslots[i].dma_pending = s->hslots[i].submitting = false;
        s->hslots[i].state = 0;
        s->hslots[i].reserved = s->hslots[i].copied = 0;
    }
    s->hcur = 0;
    s->hslots_ready = true;
    return DHSA_OK;
}

// One staged chunk: H2D from `cand`/`opp` (pinned) into the device ring on the copy stream, then
// its scan on the launch stream.  Lock held.
static int stage_and_scan_locked(dhsa_sketch *s, const uint32_t *cand, const uint32_t *opp, uint64_t cnt,
                                 cudaEvent_t also_record, int *buf_out)
{
    const int b = (int)(s->stage_seq % kStageBufs);
    if (s->stage_seq >= (uint64_t)kStageBufs) CU(cudaStreamWaitEvent(s->copy_stream, s->ev_scanned[b], 0));
    CU(cudaMemcpyAsync(s->stage_cand[b], cand, cnt * 4, cudaMemcpyHostToDevice, s->copy_stream));
    CU(cudaMemcpyAsync(s->stage_opp[b], opp, cnt * 4, cudaMemcpyHostToDevice, s->copy_stream));
    CU(cudaEventRecord(s->ev_copied[b], s->copy_stream));
    if (also_record) CU(cudaEventRecord(also_record, s->copy_stream));
    CU(cudaStreamWaitEvent(s->stream, s->ev_copied[b], 0));
    if (int rc = scan_locked(s, s->stage_cand[b], s->stage_opp[b], cnt)) return rc;
    CU(cudaEventRecord(s->ev_scanned[b], s->stream));
    s->stage_seq++;
    if (buf_out) *buf_out = b;
    return DHSA_OK;
}

// Queue one closed, completely filled slot: H2D + scan.  mu held, h.submitting set by the caller.
static int submit_slot_locked(dhsa_sketch *s, HostSlot &h)
{
    int rc = ensure_staging(s);
    if (rc == DHSA_OK) rc = stage_and_scan_locked(s, h.cand, h.opp, h.reserved, h.dma_done, nullptr);
    {
        std::lock_guard<std::mutex> lk(s->hmu);
        h.state = 0;
        h.dma_pending = rc == DHSA_OK;
        h.submitting = false;
        h.reserved = h.copied = 0;
    }
    s->hcv.notify_all();
    return rc;
}

// Everything host callers have handed over so far is queued on the launch stream when this
// returns (mu held).  Closes the partly filled slot, waits for writers still copying into closed
// slots -- they need no sketch lock for that -- and queues every slot that is ready.
static int flush_host_locked(dhsa_sketch *s)
{
    if (!s->hslots_ready) return DHSA_OK;
    std::unique_lock<std::mutex> lk(s->hmu);
    HostSlot &cur = s->hslots[s->hcur];
    if (cur.state == 1) {
        if (cur.reserved > 0) {
            cur.state = 2;
            s->hcur = (s->hcur + 1) % kHostSlots;
        } else {
            cur.state = 0;
        }
    }
    int rc = DHSA_OK;
    for (;;) {
        bool waiting = false;
        for (int i = 0; i < kHostSlots; i++) {
            HostSlot &h = s->hslots[i];
            if (h.state != 2) continue;
            if (h.copied == h.reserved && !h.submitting) {
                h.submitting = true;
                lk.unlock();
                const int r2 = submit_slot_locked(s, h);
                if (rc == DHSA_OK) rc = r2;
                lk.lock();
            } else {
                waiting = true;
            }
        }
        if (!waiting) break;
        s->hcv.wait(lk);
    }
    return rc;
}

// Host arrays through the accumulation slots.  The caller's arrays are no longer needed once
// their last byte sits in a slot; the scan itself is queued when the slot fills up or at the
// next barrier / read-out (flush_host_locked).  Called without the sketch lock, from any number
// of threads (pkg/src/dhsa/engine.py:81-86 submits batches from a pool onto one sketch).
static int update_host_ring(dhsa_sketch *s, const uint32_t *cand_host, const uint32_t *opp_host, uint64_t n)
{
    if (int rc = ensure_host_slots(s)) return rc;
    for (uint64_t off = 0; off < n;) {
        HostSlot *hp = nullptr;
        uint64_t at = 0, take = 0;
        {
            std::unique_lock<std::mutex> lk(s->hmu);
            for (;;) {
                HostSlot &h = s->hslots[s->hcur];
                if (h.state == 0 && !h.submitting) {
                    if (h.dma_pending) {  // the copy out of this slot (kHostSlots - 1 slots ago) must be over
                        if (cudaEventSynchronize(h.dma_done) != cudaSuccess) return cuda_fail(cudaGetLastError(), "host slot wait");
                        h.dma_pending = false;
                    }
                    h.state = 1;
                    h.reserved = h.copied = 0;
                }
                if (h.state == 1) break;
                s->hcv.wait(lk);  // the ring is full: wait for a slot to be queued
            }
            hp = &s->hslots[s->hcur];
            at = hp->reserved;
            take = n - off < kHostSlotPackets - at ? n - off : kHostSlotPackets - at;
            hp->reserved += take;
            if (hp->reserved == kHostSlotPackets) {
                hp->state = 2;
                s->hcur = (s->hcur + 1) % kHostSlots;
            }
        }
        CopyPool::get().copy2(hp->cand + at, cand_host + off, hp->opp + at, opp_host + off, take * 4);
        bool ready;
        {
            std::lock_guard<std::mutex> lk(s->hmu);
            hp->copied += take;
            ready = hp->state == 2 && hp->copied == hp->reserved && !hp->submitting;
        }
        s->hcv.notify_all();
        off += take;
        if (ready) {  // the writer that completes a closed slot queues it
            std::lock_guard<std::mutex> lk(s->mu);
            {
                std::lock_guard<std::mutex> hl(s->hmu);
                ready = hp->state == 2 && hp->copied == hp->reserved && !hp->submitting && hp->reserved > 0;
                if (ready) hp->submitting = true;
            }
            if (ready) {
                s->mutation_seq++;
                if (int rc = submit_slot_locked(s, *hp)) return rc;
            }
        }
    }
    return DHSA_OK;
}

// Host packets -> pinned slots / pinned caller memory -> HBM staging ring -> scan.  Copies run on
// their own stream and overlap the scan of the previous chunk.  Large page-locked arrays are DMA'd
// in place (the call returns once their last byte has been read); everything else -- ordinary
// numpy arrays, small batches -- is appended to the accumulation slots.
extern "C" int dhsa_update_host(dhsa_sketch_t *s, const uint32_t *cand_host, const uint32_t *opp_host, uint64_t n)
{
    NEED(s);
    if (n == 0) return DHSA_OK;
    NEED(cand_host);
    NEED(opp_host);
    if (int rc = use_device(s)) return rc;
    if (n < kHostSlotPackets || is_pageable(cand_host) || is_pageable(opp_host))
        return update_host_ring(s, cand_host, opp_host, n);
    std::lock_guard<std::mutex> lk(s->mu);
    s->mutation_seq++;
    if (int rc = ensure_staging(s)) return rc;
    int last = -1;
    for (uint64_t off = 0; off < n; off += kStagePackets) {
        const uint64_t cnt = (n - off < kStagePackets) ? (n - off) : kStagePackets;
        if (int rc = stage_and_scan_locked(s, cand_host + off, opp_host + off, cnt, nullptr, &last)) return rc;
    }
    if (last >= 0) CU(cudaEventSynchronize(s->ev_copied[last]));
    return DHSA_OK;
}

extern "C" int dhsa_seal(dhsa_sketch_t *s)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

extern "C" int dhsa_download_bits(dhsa_sketch_t *s, uint8_t *bits_host, uint64_t nbytes)
{
    NEED(s);
    NEED(bits_host);
    if (nbytes != s->nbytes) return fail(DHSA_EDATA, "bits buffer is %llu bytes, sketch holds %llu",
                                         (unsigned long long)nbytes, (unsigned long long)s->nbytes);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    CU(cudaMemcpyAsync(bits_host, s->bits, nbytes, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

// A byte range of the bit array, for callers that stream a sketch to or from a file in pieces
// (snapshots) instead of holding a second whole copy on the host.
extern "C" int dhsa_download_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t nbytes, uint8_t *dst_host)
{
    NEED(s);
    if (nbytes == 0) return DHSA_OK;
    NEED(dst_host);
    if (byte_lo > s->nbytes || nbytes > s->nbytes - byte_lo)
        return fail(DHSA_EDATA, "range [%llu, +%llu) outside the sketch's %llu bytes", (unsigned long long)byte_lo,
                    (unsigned long long)nbytes, (unsigned long long)s->nbytes);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    CU(cudaMemcpyAsync(dst_host, s->bits + byte_lo, nbytes, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

extern "C" int dhsa_upload_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t nbytes, const uint8_t *src_host)
{
    NEED(s);
    if (nbytes == 0) return DHSA_OK;
    NEED(src_host);
    if (byte_lo > s->nbytes || nbytes > s->nbytes - byte_lo)
        return fail(DHSA_EDATA, "range [%llu, +%llu) outside the sketch's %llu bytes", (unsigned long long)byte_lo,
                    (unsigned long long)nbytes, (unsigned long long)s->nbytes);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    s->mutation_seq++;
    CU(cudaMemcpyAsync(s->bits + byte_lo, src_host, nbytes, cudaMemcpyHostToDevice, s->stream));
    if (int rc = clear_flow_cache_locked(s, true)) return rc;  // bits may have disappeared
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

extern "C" int dhsa_download_cell(dhsa_sketch_t *s, int32_t array, uint64_t index, uint8_t *cell_host, uint64_t nbytes)
{
    NEED(s);
    NEED(cell_host);
    const uint64_t cell_bytes = (uint64_t)s->params.g / 8;
    if (array < 0 || array >= s->params.r || index >= (1ull << s->params.k))
        return fail(DHSA_ECONFIG, "estimator (%d, %llu) outside the sketch's %d x 2^%d cells", array,
                    (unsigned long long)index, s->params.r, s->params.k);
    if (nbytes != cell_bytes) return fail(DHSA_EDATA, "cell buffer is %llu bytes, an estimator holds %llu",
                                          (unsigned long long)nbytes, (unsigned long long)cell_bytes);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    const uint64_t off = (((uint64_t)array << s->params.k) + index) * cell_bytes;
    CU(cudaMemcpyAsync(cell_host, s->bits + off, cell_bytes, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

extern "C" int dhsa_upload_bits(dhsa_sketch_t *s, const uint8_t *bits_host, uint64_t nbytes)
{
    NEED(s);
    NEED(bits_host);
    if (nbytes != s->nbytes) return fail(DHSA_EDATA, "bits buffer is %llu bytes, sketch holds %llu",
                                         (unsigned long long)nbytes, (unsigned long long)s->nbytes);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    s->mutation_seq++;
    CU(cudaMemcpyAsync(s->bits, bits_host, nbytes, cudaMemcpyHostToDevice, s->stream));
    if (int rc = clear_flow_cache_locked(s, true)) return rc;
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

// ---------------------------------------------------------------- read-out --

static int ensure_readout(dhsa_sketch *s)
{
    if (s->lists) return DHSA_OK;
    CU(cudaMalloc(&s->lists, s->dp.ncell * sizeof(uint32_t)));
    CU(cudaMalloc(&s->bitmaps, (uint64_t)s->params.r * s->bitmap_words * sizeof(uint32_t)));
    return DHSA_OK;
}

static int ensure_host_tmp(dhsa_sketch *s, uint64_t bytes)
{
    if (bytes <= s->host_tmp_bytes) return DHSA_OK;
    if (s->host_tmp) cudaFreeHost(s->host_tmp);
    s->host_tmp = nullptr, s->host_tmp_bytes = 0;
    CU(cudaMallocHost(&s->host_tmp, bytes));
    s->host_tmp_bytes = bytes;
    return DHSA_OK;
}

static uint64_t pow2_at_least(uint64_t v)
{
    uint64_t l = 1;
    while (l < v) l <<= 1;
    return l;
}

// Workspaces of the stage chain: 64 bytes per partial key.  max_candidates is only a bound in the
// reference (pkg/src/dhsa/dhla.py:34,269-273), and callers pass huge values for "unlimited", so the
// buffers start at the default bound and grow when a stage needs more (restore_collect).
static uint64_t initial_candidates()
{
    static const uint64_t v = [] {
        uint64_t n = 1ull << 20;  // DEFAULT_MAX_CANDIDATES, dhla.py:34
        if (const char *env = getenv("DHSA_INITIAL_CANDIDATES")) {  // tests shrink it to exercise the growth path
            const long long q = strtoll(env, nullptr, 10);
            if (q >= 1) n = (uint64_t)q;
        }
        return n;
    }();
    return v;
}

static int ensure_candidates(dhsa_sketch *s, uint64_t want)
{
    if (want < 1) want = 1;
    if (want <= s->cand_cap) return DHSA_OK;
    CU(cudaStreamSynchronize(s->stream));
    for (int b = 0; b < 2; b++) {
        cudaFree(s->sub[b]);
        cudaFree(s->cl0[b]);
        s->sub[b] = nullptr, s->cl0[b] = nullptr;
    }
    cudaFree(s->keys);
    cudaFree(s->cand_sz);
    cudaFree(s->packed);
    cudaFree(s->reports);
    s->keys = nullptr, s->packed = nullptr, s->reports = nullptr, s->cand_sz = nullptr;
    s->cand_cap = 0;
    for (int b = 0; b < 2; b++) {
        CU(cudaMalloc(&s->sub[b], want * sizeof(uint64_t)));
        CU(cudaMalloc(&s->cl0[b], want * sizeof(uint32_t)));
    }
    s->packed_cap = pow2_at_least(want);
    CU(cudaMalloc(&s->keys, s->packed_cap * sizeof(uint64_t)));
    CU(cudaMalloc(&s->cand_sz, want * sizeof(int32_t)));
    CU(cudaMalloc(&s->packed, s->packed_cap * sizeof(uint64_t)));
    CU(cudaMalloc(&s->reports, want * sizeof(ReportOut)));
    s->cand_cap = want;
    return DHSA_OK;
}

// entries the stage buffers hold for a read-out bounded by max_candidates
static uint64_t buffer_cap(const dhsa_sketch *s, uint64_t max_candidates)
{
    return max_candidates < s->cand_cap ? max_candidates : s->cand_cap;
}

static int ensure_candidates_for(dhsa_sketch *s, uint64_t max_candidates)
{
    const uint64_t first = initial_candidates();
    if (s->cand_cap >= max_candidates || s->cand_cap >= first) return DHSA_OK;
    return ensure_candidates(s, max_candidates < first ? max_candidates : first);
}

// K2: zero counts of the cells [cell_lo, cell_hi) -- every cell, or this rank's range of a partitioned read-out.
static int launch_zero_counts(dhsa_sketch *s, uint64_t cell_lo, uint64_t cell_hi)
{
    if (cell_lo >= cell_hi) return DHSA_OK;
    const uint64_t bpe = (uint64_t)s->params.g / 8, ncell = cell_hi - cell_lo;
    const uint8_t *first = s->bits + cell_lo * bpe;
    if (bpe >= 16) {
        const int vecs = (int)(bpe / 16);
        const int lanes = vecs < 32 ? vecs : 32;
        const int grid = grid_for(s, ncell * (uint64_t)lanes, 256, 8);
        k_zero_counts_vec<<<grid, 256, 0, s->stream>>>(reinterpret_cast<const uint4 *>(first), s->zc + cell_lo, ncell,
                                                       vecs, lanes, s->params.g);
    } else {
        const int grid = grid_for(s, ncell, 256, 8);
        k_zero_counts_small<<<grid, 256, 0, s->stream>>>(first, s->zc + cell_lo, ncell, (int)bpe, s->params.g);
    }
    s->launches++;
    CU(cudaGetLastError());
    return DHSA_OK;
}

static int refuse_if_restore_pending(const dhsa_sketch *s);

// ---- the read-out's floating point, on the host -----------------------------------------------
// Every number the reference derives with float64 math is derived here with the same formula and
// the host's libm, as the reference does (math.log / math.exp / ** on Python floats):
//   zmin        = g exp(-theta / g)                                  dhla.py:45-47
//   flow count  = mean_i( -C ln(ZR(i)/C) ), ZR == 0 -> 1, saturated  estimator.py:26-34, dhla.py:121-128
//   psi         = 1 - exp(-flow / C)                                 dhla.py:130-134
//   denom       = g (1 - psi^r)                                      dhla.py:184
//   estimate    = -g ln(SZ'/denom), 0.0 when SZ' >= denom            dhla.py:183-189
// and the two threshold decisions become integer compares the kernels apply exactly:
//   hot   <=> zc < zmin          <=> zc <= zc_cut    (zc_cut = the largest integer below zmin)
//   keep  <=> estimate >= theta  <=> SZ' <= sz_cut   (the estimate is non-increasing in SZ')
// zc_cut is known before the read-out is queued.  sz_cut needs psi, i.e. the zero totals the device
// is about to count, so the device bisects its own cut (report_cut) to keep the chain free of host
// round trips, and the host recomputes it here from the zero totals that came back: if the two ever
// differ, the reports are re-filtered on the device with the host's cut (restore_collect).
static int hot_cut(const dhsa_sketch *s, double theta)
{
    const double g = (double)s->params.g;
    const double zmin = g * exp(-theta / g);
    if (!(zmin > 0.0)) return -1;                     // nothing is below zero (also NaN)
    if (zmin > g) return s->params.g;                 // theta < 0: every cell is hot
    long long c = (long long)ceil(zmin) - 1;          // largest integer strictly below zmin
    while ((double)(c + 1) < zmin) c++;
    while (c >= 0 && !((double)c < zmin)) c--;
    return (int)c;
}

struct HostScalars {
    double flow, psi, denom;
    int flow_saturated;
    int sz_cut;
};

static double host_estimate(int g, long long sz_clamped, double denom)
{
    if ((double)sz_clamped >= denom) return 0.0;
    return -(double)g * log((double)sz_clamped / denom);
}

static HostScalars host_scalars(const dhsa_sketch *s, const long long *zero_totals, double theta)
{
    HostScalars h;
    const int r = s->params.r, g = s->params.g;
    const double cap = (double)g * (double)(1ull << s->params.k);
    // sum(e.value for e in per_array) (dhla.py:127): the interpreter this reference runs on (CPython >= 3.12)
    // adds floats with Neumaier's compensated summation, so the mean is formed the same way here --
    // the last bit of the flow count would otherwise differ from the live reference's
    double acc = 0.0, comp = 0.0;
    h.flow_saturated = 0;
    for (int i = 0; i < r; i++) {
        long long z = zero_totals[i];
        if (z == 0) {
            h.flow_saturated = 1;
            z = 1;
        }
        const double x = -cap * log((double)z / cap);
        const double t = acc + x;
        comp += fabs(acc) >= fabs(x) ? (acc - t) + x : (x - t) + acc;
        acc = t;
    }
    if (comp != 0.0 && isfinite(comp)) acc += comp;
    h.flow = acc / r;
    h.psi = 1.0 - exp(-h.flow / cap);
    h.denom = g * (1.0 - pow(h.psi, (double)r));
    // largest SZ' in [1, g] whose estimate reaches theta (0 = none): bisection, then a walk over the
    // neighbours so that a non-monotone last bit of log() cannot leave the boundary one step off
    int cut = 0;
    if (host_estimate(g, 1, h.denom) >= theta) {
        int lo = 1, hi = g;
        if (host_estimate(g, hi, h.denom) >= theta) {
            lo = hi;
        } else {
            while (hi - lo > 1) {
                const int mid = lo + ((hi - lo) >> 1);
                if (host_estimate(g, mid, h.denom) >= theta) lo = mid; else hi = mid;
            }
        }
        while (lo < g && host_estimate(g, lo + 1, h.denom) >= theta) lo++;
        cut = lo;
    }
    h.sz_cut = cut;
    return h;
}

// K2 + hot sets + scalars, stream-ordered.
static int launch_estimate(dhsa_sketch *s, double theta)
{
    if (int rc = ensure_readout(s)) return rc;
    if (s->zc_given) {
        s->zc_given = false;  // the caller's zero counts are already in s->zc (dhsa_use_zero_counts)
    } else if (s->owners.n > 0) {
        // partitioned read-out: s->zc was counted range by range on the owners and gathered (multi.py)
    } else if (int rc = launch_zero_counts(s, 0, s->dp.ncell)) {
        return rc;
    }
    k_hot_sets<<<s->params.r, 1024, 0, s->stream>>>(s->zc, hot_cut(s, theta), theta, s->params.r, s->params.k,
                                                   s->params.g, s->lists, s->bitmaps, s->bitmap_words, s->ctl);
    s->launches += 1;
    CU(cudaGetLastError());
    return DHSA_OK;
}

// K3: stage chain -> verified keys in s->keys, count in ctl->n_candidates.
static int launch_restore_stages(dhsa_sketch *s, uint64_t max_candidates, bool verify, int *last_buf)
{
    const uint64_t cap = buffer_cap(s, max_candidates);
    const int r = s->params.r, n_stages = r - 2;
    const int grid = s->sm_count * DHSA_READOUT_CTAS_PER_SM;
    k_stage_first<<<grid, 256, 0, s->stream>>>(s->lists, s->bitmaps, s->bitmap_words, s->dp, cap, s->sub[0], s->cl0[0],
                                               s->ctl);
    int cur = 0;
    for (int i = 3; i < r; i++) {
        k_stage_next<<<grid, 256, 0, s->stream>>>(i, s->lists, s->bitmaps, s->bitmap_words, s->dp, cap, s->sub[cur],
                                                  s->cl0[cur], s->sub[cur ^ 1], s->cl0[cur ^ 1], s->ctl);
        cur ^= 1;
    }
    if (verify)
        k_verify_keys<<<grid, 256, 0, s->stream>>>(n_stages, s->dp, cap, max_candidates, s->sub[cur], s->cl0[cur], s->keys,
                                                   s->ctl);
    if (last_buf) *last_buf = cur;
    s->launches += (uint64_t)n_stages + (verify ? 1 : 0);
    CU(cudaGetLastError());
    return DHSA_OK;
}

static int read_control(dhsa_sketch *s)
{
    CU(cudaMemcpyAsync(s->ctl_host, s->ctl, sizeof(Control), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

// Host-driven bitonic sort for more than DHSA_SORT_SMEM_MAX entries.
static int sort_large(dhsa_sketch *s, uint64_t *data, uint64_t n)
{
    const uint64_t len = pow2_at_least(n);
    const int grid = grid_for(s, len, 256, 8);
    k_sort_pad<<<grid, 256, 0, s->stream>>>(data, n, len);
    s->launches++;
    for (uint64_t kk = 2; kk <= len; kk <<= 1)
        for (uint64_t j = kk >> 1; j > 0; j >>= 1) {
            k_bitonic_pass<<<grid, 256, 0, s->stream>>>(data, len, kk, j);
            s->launches++;
        }
    CU(cudaGetLastError());
    return DHSA_OK;
}

// *info from the control block that came back, with the float64 scalars from the host's formulas.
static void fill_info(const dhsa_sketch *s, double theta, dhsa_restore_info_t *info)
{
    if (!info) return;
    const Control *c = s->ctl_host;
    memset(info, 0, sizeof *info);
    const HostScalars h = host_scalars(s, c->zero_totals, theta);
    info->n_candidates = c->n_candidates;
    info->n_reports = c->n_reports;
    info->fail_stage = c->fail_stage;
    info->fail_count = c->fail_count;
    info->flow_saturated = h.flow_saturated;
    info->flow_count = h.flow;
    info->psi = h.psi;
    info->denom = h.denom;
    info->sz_cut = h.sz_cut;
    info->hot_cut = hot_cut(s, theta);
    for (int i = 0; i < 64; i++) {
        info->hot_counts[i] = c->hot_counts[i];
        info->stage_counts[i] = c->stage_counts[i];
        info->zero_totals[i] = c->zero_totals[i];
    }
}

extern "C" int dhsa_zero_counts(dhsa_sketch_t *s, int64_t *zc_host, int64_t *zr_host)
{
    NEED(s);
    NEED(zc_host);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    s->zc_given = false;
    if (int rc = launch_estimate(s, 0.0)) return rc;
    // widen on the host side of the copy: device keeps int32, the reference API is int64
    if (int rc = ensure_host_tmp(s, s->dp.ncell * sizeof(int32_t))) return rc;
    int32_t *tmp = static_cast<int32_t *>(s->host_tmp);
    CU(cudaMemcpyAsync(tmp, s->zc, s->dp.ncell * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(s->ctl_host, s->ctl, sizeof(Control), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (uint64_t c = 0; c < s->dp.ncell; c++) zc_host[c] = tmp[c];
    if (zr_host)
        for (int i = 0; i < s->params.r; i++) zr_host[i] = s->ctl_host->zero_totals[i];
    return DHSA_OK;
}

// The reference's read-out methods take an optional zero_counts= array and use it in place of
// counting the bits (hot_sets dhla.py:111-119, estimate_flow_count :121-128, _candidate_hosts
// :198-207).  One-shot: the next dhsa_hot_sets / dhsa_estimate / dhsa_candidate_hosts on this handle
// starts from these counts.
extern "C" int dhsa_use_zero_counts(dhsa_sketch_t *s, const int64_t *zc_host)
{
    NEED(s);
    NEED(zc_host);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = ensure_readout(s)) return rc;
    if (int rc = ensure_host_tmp(s, s->dp.ncell * sizeof(int32_t))) return rc;
    int32_t *tmp = static_cast<int32_t *>(s->host_tmp);
    for (uint64_t c = 0; c < s->dp.ncell; c++) {
        if (zc_host[c] < 0 || zc_host[c] > s->params.g)
            return fail(DHSA_EDATA, "zero count %lld of cell %llu outside [0, g=%d]", (long long)zc_host[c],
                        (unsigned long long)c, s->params.g);
        tmp[c] = (int32_t)zc_host[c];
    }
    CU(cudaMemcpyAsync(s->zc, tmp, s->dp.ncell * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
    CU(cudaStreamSynchronize(s->stream));  // host_tmp is reused by the read-out that follows
    s->zc_given = true;
    return DHSA_OK;
}

extern "C" int dhsa_hot_sets(dhsa_sketch_t *s, double theta, uint64_t *lists_host, uint64_t *counts_host)
{
    NEED(s);
    NEED(lists_host);
    NEED(counts_host);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    if (int rc = launch_estimate(s, theta)) return rc;
    if (int rc = ensure_host_tmp(s, s->dp.ncell * sizeof(uint32_t))) return rc;
    uint32_t *tmp = static_cast<uint32_t *>(s->host_tmp);
    CU(cudaMemcpyAsync(tmp, s->lists, s->dp.ncell * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream));
    if (int rc = read_control(s)) return rc;
    const uint64_t m = 1ull << s->params.k;
    for (int i = 0; i < s->params.r; i++) {
        const uint64_t n = s->ctl_host->hot_counts[i];
        counts_host[i] = n;
        for (uint64_t q = 0; q < n; q++) lists_host[(uint64_t)i * m + q] = tmp[(uint64_t)i * m + q];
    }
    return DHSA_OK;
}

extern "C" int dhsa_estimate(dhsa_sketch_t *s, double theta, dhsa_restore_info_t *info)
{
    NEED(s);
    NEED(info);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    if (int rc = launch_estimate(s, theta)) return rc;
    if (int rc = read_control(s)) return rc;
    fill_info(s, theta, info);
    return DHSA_OK;
}

static int capacity_error(const dhsa_sketch *s, uint64_t max_candidates)
{
    // text of pkg/src/dhsa/dhla.py:270-273 / 295-298
    return fail(DHSA_ECAPACITY, "restore stage %d produced %llu partial keys (max_candidates=%llu)",
                s->ctl_host->fail_stage, (unsigned long long)s->ctl_host->fail_count,
                (unsigned long long)max_candidates);
}

// The stage buffers were too small for a stage that max_candidates allows: how many entries the
// rerun needs (0 = the buffers were large enough).  ctl_host holds the control block of the run.
static uint64_t regrow_target(const dhsa_sketch *s, uint64_t max_candidates)
{
    const Control *c = s->ctl_host;
    if (c->fail_stage || c->any_empty) return 0;
    const uint64_t cap = buffer_cap(s, max_candidates);
    for (int st = 0; st < s->params.r - 2; st++)
        if (c->stage_counts[st] > cap) {
            uint64_t want = pow2_at_least(c->stage_counts[st]);
            return want < max_candidates ? want : max_candidates;
        }
    return 0;
}

extern "C" int dhsa_candidate_hosts(dhsa_sketch_t *s, double theta, uint64_t max_candidates, uint64_t *hosts_host,
                                    uint64_t hosts_cap, dhsa_restore_info_t *info)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    if (int rc = ensure_readout(s)) return rc;
    if (int rc = ensure_candidates_for(s, max_candidates)) return rc;
    const bool zc_given = s->zc_given;  // a rerun after growing the workspaces starts from the same zero counts
    for (;;) {
        s->zc_given = zc_given;
        if (int rc = launch_estimate(s, theta)) return rc;
        if (int rc = launch_restore_stages(s, max_candidates, true, nullptr)) return rc;
        k_sort_small<<<1, 1024, DHSA_SORT_SMEM_MAX * sizeof(uint64_t), s->stream>>>(s->keys, &s->ctl->n_candidates, s->ctl,
                                                                                     nullptr, 0, nullptr, nullptr);
        s->launches++;
        CU(cudaGetLastError());
        if (int rc = read_control(s)) return rc;
        const uint64_t want = regrow_target(s, max_candidates);
        if (!want) break;
        if (int rc = ensure_candidates(s, want)) return rc;  // the bits are untouched: run the chain again
    }
    fill_info(s, theta, info);
    if (s->ctl_host->fail_stage) return capacity_error(s, max_candidates);
    const uint64_t n = s->ctl_host->n_candidates;
    if (n > DHSA_SORT_SMEM_MAX)
        if (int rc = sort_large(s, s->keys, n)) return rc;
    if (n > hosts_cap) return fail(DHSA_EDATA, "%llu candidate hosts exceed the output capacity %llu",
                                   (unsigned long long)n, (unsigned long long)hosts_cap);
    if (n) {
        NEED(hosts_host);
        CU(cudaMemcpyAsync(hosts_host, s->keys, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
    }
    return DHSA_OK;
}

extern "C" int dhsa_shared_zero_counts(dhsa_sketch_t *s, const uint64_t *hosts_host, uint64_t n, int64_t *sz_host)
{
    NEED(s);
    if (n == 0) return DHSA_OK;
    NEED(hosts_host);
    NEED(sz_host);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    if (n > s->hosts_in_cap) {
        CU(cudaStreamSynchronize(s->stream));
        cudaFree(s->hosts_in);
        cudaFree(s->sz_out);
        s->hosts_in = nullptr, s->sz_out = nullptr, s->hosts_in_cap = 0;
        CU(cudaMalloc(&s->hosts_in, n * sizeof(uint64_t)));
        CU(cudaMalloc(&s->sz_out, n * sizeof(int32_t)));
        s->hosts_in_cap = n;
    }
    CU(cudaMemcpyAsync(s->hosts_in, hosts_host, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream));
    const int grid = grid_for(s, n * 32, 256, 8);
    if (s->owners.n > 0)
        k_shared_zero_counts_owned<<<grid, 256, 0, s->stream>>>(s->owners, s->dp, s->hosts_in, n, s->sz_out);
    else
        k_shared_zero_counts<<<grid, 256, 0, s->stream>>>(s->bits, s->dp, s->hosts_in, n, s->sz_out);
    s->launches++;
    CU(cudaGetLastError());
    int32_t *tmp = (int32_t *)malloc(n * sizeof(int32_t));
    if (!tmp) return fail(-1, "out of host memory");
    cudaError_t e = cudaMemcpyAsync(tmp, s->sz_out, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) {
        free(tmp);
        return cuda_fail(e, "shared_zero_counts readback");
    }
    for (uint64_t t = 0; t < n; t++) sz_host[t] = tmp[t];
    free(tmp);
    return DHSA_OK;
}

// The whole read-out -- zero counts, hot sets + scalars, stage chain, verify, re-estimate, sort,
// emit, and the copy-back of the control block and the first kPinnedReports rows -- enqueued on
// s->stream.  Called directly, or once under stream capture to build the graph.
static int enqueue_restore(dhsa_sketch *s, double theta, uint64_t max_candidates)
{
    if (int rc = launch_estimate(s, theta)) return rc;
    int cur = 0;
    if (int rc = launch_restore_stages(s, max_candidates, false, &cur)) return rc;
    const int grid = s->sm_count * DHSA_READOUT_CTAS_PER_SM;
    // verify + re-estimate, then sort + emit: two launches for what were four
    if (s->owners.n > 0)
        k_verify_reestimate_owned<<<grid, 256, 0, s->stream>>>(s->params.r - 2, s->dp, buffer_cap(s, max_candidates),
                                                               max_candidates, s->sub[cur], s->cl0[cur], s->owners, s->keys,
                                                               s->cand_sz, s->packed, s->ctl);
    else
        k_verify_reestimate<<<grid, 256, 0, s->stream>>>(s->params.r - 2, s->dp, buffer_cap(s, max_candidates),
                                                         max_candidates, s->sub[cur], s->cl0[cur], s->bits, s->keys,
                                                         s->cand_sz, s->packed, s->ctl);
    // sort + emit; as the last kernel it also gathers the window counters (6 words behind the bit array) and
    // the first report rows behind the control block: ONE copy brings everything the host reads back
    k_sort_small<<<1, 1024, DHSA_SORT_SMEM_MAX * sizeof(uint64_t), s->stream>>>(
        s->packed, &s->ctl->n_reports, s->ctl, s->reports, s->params.g, s->tally, s->rb->head);
    s->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(s->rb_host, s->rb, sizeof(Readback), cudaMemcpyDeviceToHost, s->stream));
    return DHSA_OK;
}

// One graph launch instead of eight kernel launches and two copies: the chain is latency-bound
// (every kernel is microseconds), so launch gaps are a third of its time.  Falls back to direct
// launches if capture is not possible on the current stream (same kernels either way).
static int run_restore(dhsa_sketch *s, double theta, uint64_t max_candidates)
{
    if (int rc = ensure_readout(s)) return rc;
    if (int rc = ensure_candidates_for(s, max_candidates)) return rc;
    if (!s->graph_disabled) {
        const bool fresh = s->restore_graph && s->graph_theta == theta && s->graph_owners_seq == s->owners_seq &&
                           s->graph_max_candidates == max_candidates && s->graph_cand_cap == s->cand_cap;
        if (!fresh) {
            if (s->restore_graph) {
                cudaGraphExecDestroy(s->restore_graph);
                s->restore_graph = nullptr;
            }
            const uint64_t before = s->launches;
            cudaGraph_t graph = nullptr;
            // captured on the sketch's own stream (the caller's may be the legacy default stream, which
            // cannot capture); the instantiated graph launches on whatever stream the sketch uses
            cudaStream_t launch_stream = s->stream;
            s->stream = s->own_stream;
            cudaError_t e = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                const int rc = enqueue_restore(s, theta, max_candidates);
                e = cudaStreamEndCapture(s->stream, &graph);
                if (rc != DHSA_OK && e == cudaSuccess) e = cudaErrorUnknown;
            }
            s->stream = launch_stream;
            if (e == cudaSuccess) e = cudaGraphInstantiate(&s->restore_graph, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            s->graph_kernels = s->launches - before;
            s->launches = before;
            if (e != cudaSuccess) {
                (void)cudaGetLastError();
                s->restore_graph = nullptr;
                s->graph_disabled = true;  // e.g. the caller's stream is itself being captured
            } else {
                s->graph_theta = theta;
                s->graph_max_candidates = max_candidates;
                s->graph_cand_cap = s->cand_cap;
                s->graph_owners_seq = s->owners_seq;
            }
        }
        if (s->restore_graph) {
            CU(cudaGraphLaunch(s->restore_graph, s->stream));
            s->launches += s->graph_kernels;
            return DHSA_OK;
        }
    }
    return enqueue_restore(s, theta, max_candidates);
}

// A read-out call that uses the pinned mirrors while a begun restore has not been collected
static int refuse_if_restore_pending(const dhsa_sketch *s)
{
    if (s->restore_pending)
        return fail(DHSA_ECONFIG, "a restore begun with dhsa_restore_begin has not been collected with dhsa_restore_end");
    return DHSA_OK;
}

static int restore_begin_locked(dhsa_sketch *s, double theta, uint64_t max_candidates)
{
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    s->zc_given = false;  // restore_superpoints always counts the bits itself (dhla.py:176)
    if (int rc = run_restore(s, theta, max_candidates)) return rc;
    CU(cudaEventRecord(s->restore_ev, s->stream));
    s->restore_pending = true;
    s->restore_max_candidates = max_candidates;
    s->restore_theta = theta;
    s->restore_seq = s->mutation_seq;
    return DHSA_OK;
}

// The filter and the sort again with the host's scalars (denom, sz_cut) in the device control
// block -- taken when the device's own libm put the cut, or the zero-estimate class, one step away
// from where the host's formulas put it.  Uses only what the read-out left in the workspaces (the
// verified keys and their SZ), not the bits: the next window may already be in them.
static int refilter_with_host_cut(dhsa_sketch *s, const HostScalars &h)
{
    Control *c = s->ctl_host;
    c->denom = h.denom, c->psi = h.psi, c->flow_count = h.flow;
    c->n_reports = 0;
    c->sorted = 0;
    CU(cudaMemcpyAsync(s->ctl, c, sizeof(Control), cudaMemcpyHostToDevice, s->stream));
    const int grid = s->sm_count * DHSA_READOUT_CTAS_PER_SM;
    k_refilter<<<grid, 256, 0, s->stream>>>(s->keys, s->cand_sz, h.sz_cut, s->packed, s->ctl);
    k_sort_small<<<1, 1024, DHSA_SORT_SMEM_MAX * sizeof(uint64_t), s->stream>>>(
        s->packed, &s->ctl->n_reports, s->ctl, s->reports, s->params.g, nullptr, s->rb->head);
    s->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(s->rb_host, s->rb, sizeof(Readback), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return DHSA_OK;
}

static int restore_end_locked(dhsa_sketch *s, dhsa_report_t *reports_host, uint64_t reports_cap,
                              dhsa_restore_info_t *info)
{
    if (!s->restore_pending) return fail(DHSA_ECONFIG, "dhsa_restore_end without dhsa_restore_begin");
    CU(cudaEventSynchronize(s->restore_ev));
    // the window's flow-cache counters came back with the control block: the auto policy's prior for the next long
    // launch (a pipelined caller resets before the side-stream snapshot has landed, and reset drops it)
    if (s->scan_mode == DHSA_SCAN_AUTO && s->ctl_host->counters[2] >= kPolicyMinSample)
        s->auto_cache_trusted = !projected_no_repeats(s->ctl_host->counters[2], s->ctl_host->counters[3]);
    const uint64_t max_candidates = s->restore_max_candidates;
    const double theta = s->restore_theta;
    // a stage needed more room than the workspaces had (and max_candidates allows it): grow, run again
    for (uint64_t want; (want = regrow_target(s, max_candidates)) != 0;) {
        if (s->restore_seq != s->mutation_seq) {
            s->restore_pending = false;
            return fail(DHSA_ECONFIG, "restore needs room for %llu partial keys (workspace %llu) but the sketch was modified "
                        "after dhsa_restore_begin; use dhsa_restore, or collect before the next window is fed",
                        (unsigned long long)want, (unsigned long long)s->cand_cap);
        }
        if (int rc = ensure_candidates(s, want)) return rc;
        if (int rc = run_restore(s, theta, max_candidates)) return rc;
        CU(cudaStreamSynchronize(s->stream));
    }
    if (s->ctl_host->fail_stage) {
        s->restore_pending = false;
        fill_info(s, theta, info);
        return capacity_error(s, max_candidates);
    }
    // the threshold decision belongs to the host's formulas (see host_scalars)
    const HostScalars h = host_scalars(s, s->ctl_host->zero_totals, theta);
    if (!s->ctl_host->any_empty && s->ctl_host->n_candidates &&
        (h.sz_cut != s->ctl_host->sz_cut || ceil(h.denom) != ceil(s->ctl_host->denom))) {
        if (int rc = refilter_with_host_cut(s, h)) return rc;
    }
    const int grid = s->sm_count * DHSA_READOUT_CTAS_PER_SM;
    const uint64_t n = s->ctl_host->n_reports;
    fill_info(s, theta, info);
    // too small an output buffer: the read-out stays collectable, the caller retries with n_reports rows
    if (n > reports_cap) return fail(DHSA_EDATA, "%llu reports exceed the output capacity %llu",
                                     (unsigned long long)n, (unsigned long long)reports_cap);
    s->restore_pending = false;
    bool in_pinned = n <= kPinnedReports;
    if (n > DHSA_SORT_SMEM_MAX) {  // rare: the single-CTA sorter declined, sort with global passes and re-emit
        if (int rc = sort_large(s, s->packed, n)) return rc;
        k_emit_reports<<<grid, 256, 0, s->stream>>>(s->packed, s->params.g, s->reports, s->ctl);
        s->launches++;
        CU(cudaGetLastError());
        in_pinned = false;
    }
    if (n) {
        NEED(reports_host);
        static_assert(sizeof(ReportOut) == sizeof(dhsa_report_t), "report layouts must match");
        if (in_pinned) {
            memcpy(reports_host, s->reports_pinned, n * sizeof(ReportOut));
        } else {
            CU(cudaMemcpyAsync(reports_host, s->reports, n * sizeof(ReportOut), cudaMemcpyDeviceToHost, s->stream));
            CU(cudaStreamSynchronize(s->stream));
        }
        // estimates from the integer SZ with the host's formula (the device rows carry its own libm's value)
        for (uint64_t t = 0; t < n; t++) {
            const int32_t sz = reports_host[t].shared_zero_count;
            reports_host[t].estimate = sz < 0 ? 0.0 : host_estimate(s->params.g, sz == 0 ? 1 : sz, h.denom);
        }
    }
    return DHSA_OK;
}

extern "C" int dhsa_restore(dhsa_sketch_t *s, double theta, uint64_t max_candidates, dhsa_report_t *reports_host,
                            uint64_t reports_cap, dhsa_restore_info_t *info)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = restore_begin_locked(s, theta, max_candidates)) return rc;
    const int rc = restore_end_locked(s, reports_host, reports_cap, info);
    s->restore_pending = false;  // one call: a too-small buffer is reported, not kept pending
    return rc;
}

extern "C" int dhsa_restore_begin(dhsa_sketch_t *s, double theta, uint64_t max_candidates)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    return restore_begin_locked(s, theta, max_candidates);
}

extern "C" int dhsa_restore_end(dhsa_sketch_t *s, dhsa_report_t *reports_host, uint64_t reports_cap,
                                dhsa_restore_info_t *info)
{
    NEED(s);
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    return restore_end_locked(s, reports_host, reports_cap, info);
}

// ------------------------------------------------------- hash group, stateless --

static int dev_params_from(const dhsa_params_t *params, DevParams *d)
{
    if (int rc = validate(params)) return rc;
    memset(d, 0, sizeof *d);
    const uint64_t m = 1ull << params->k;
    d->r = params->r, d->k = params->k, d->alpha = params->alpha, d->key_width = params->key_width;
    d->log2g = ilog2_exact(params->g);
    d->kmask = (uint32_t)(m - 1);
    d->gmask = (uint32_t)(params->g - 1);
    d->state_dh0 = params->state_dh0, d->state_h1 = params->state_h1;
    d->ncell = (uint64_t)params->r * m;
    return DHSA_OK;
}

// shared body of the two calls below: `in` (n x in_width u64) -> out0 (n x out_width u64) [+ ok bytes]
static int hash_group_call(const dhsa_params_t *params, int device, bool inverse, const uint64_t *in_host, uint64_t n,
                           uint64_t *out_host, uint8_t *ok_host)
{
    NEED(params);
    DevParams d;
    if (int rc = dev_params_from(params, &d)) return rc;
    if (n == 0) return DHSA_OK;
    NEED(in_host);
    NEED(out_host);
    if (inverse) NEED(ok_host);
    CU(cudaSetDevice(device));
    const uint64_t in_w = inverse ? (uint64_t)d.r : 1, out_w = inverse ? 1 : (uint64_t)d.r;
    uint64_t *in_dev = nullptr, *out_dev = nullptr;
    uint8_t *ok_dev = nullptr;
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&in_dev, n * in_w * 8);
    if (e == cudaSuccess) e = cudaMalloc(&out_dev, n * out_w * 8);
    if (e == cudaSuccess && inverse) e = cudaMalloc(&ok_dev, n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(in_dev, in_host, n * in_w * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        int sms = 1;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        uint64_t want = (n + 255) / 256, cap = (uint64_t)sms * 8;
        const int grid = (int)(want < cap ? want : cap);
        if (inverse)
            k_reconstruct_many<<<grid, 256, 0, st>>>(d, in_dev, n, out_dev, ok_dev);
        else
            k_forward_many<<<grid, 256, 0, st>>>(d, in_dev, n, out_dev);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, out_dev, n * out_w * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && inverse) e = cudaMemcpyAsync(ok_host, ok_dev, n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(in_dev), cudaFree(out_dev), cudaFree(ok_dev);
    if (st) cudaStreamDestroy(st);
    if (e != cudaSuccess) return cuda_fail(e, inverse ? "reconstruct_many" : "forward_many");
    return DHSA_OK;
}

extern "C" int dhsa_forward_many(const dhsa_params_t *params, int device, const uint64_t *keys_host, uint64_t n,
                                 uint64_t *indices_host)
{
    return hash_group_call(params, device, false, keys_host, n, indices_host, nullptr);
}

extern "C" int dhsa_reconstruct_many(const dhsa_params_t *params, int device, const uint64_t *tuples_host, uint64_t n,
                                     uint64_t *keys_host, uint8_t *ok_host)
{
    return hash_group_call(params, device, true, tuples_host, n, keys_host, ok_host);
}

// ------------------------------------------------------------------- merge --

static int same_params(const dhsa_sketch *a, const dhsa_sketch *b)
{
    const dhsa_params_t &x = a->params, &y = b->params;
    if (x.r != y.r || x.g != y.g || x.k != y.k || x.alpha != y.alpha || x.key_width != y.key_width ||
        x.state_dh0 != y.state_dh0 || x.state_h1 != y.state_h1)
        return fail(DHSA_ECONFIG, "cannot merge sketches with different parameters");
    return DHSA_OK;
}

static int merge_range_locked(dhsa_sketch *dst, const void *const *peers, int n_peers, uint64_t byte_lo,
                              uint64_t byte_hi)
{
    if (n_peers < 1 || n_peers > DHSA_MAX_PEERS)
        return fail(DHSA_ECONFIG, "n_peers must be in [1, %d] (got %d)", DHSA_MAX_PEERS, n_peers);
    if ((byte_lo | byte_hi) & 15u) return fail(DHSA_ECONFIG, "merge range must be 16-byte aligned");
    if (byte_lo > byte_hi || byte_hi > dst->alloc_bytes) return fail(DHSA_ECONFIG, "merge range out of bounds");
    if (byte_lo == byte_hi) return DHSA_OK;
    PeerPtrs pp;
    for (int q = 0; q < DHSA_MAX_PEERS; q++) pp.p[q] = q < n_peers ? reinterpret_cast<const uint4 *>(peers[q]) : nullptr;
    const uint64_t lo = byte_lo / 16, hi = byte_hi / 16;
    const int grid = grid_for(dst, hi - lo, 256, 8);
    k_or_merge<<<grid, 256, 0, dst->stream>>>(reinterpret_cast<uint4 *>(dst->bits), pp, n_peers, lo, hi);
    dst->launches++;
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_or_merge(dhsa_sketch_t *dst, dhsa_sketch_t *src)
{
    NEED(dst);
    NEED(src);
    if (int rc = same_params(dst, src)) return rc;
    if (dst == src) return DHSA_OK;
    // src's pending updates must land before dst reads them
    {
        std::lock_guard<std::mutex> lk(src->mu);
        if (int rc = use_device(src)) return rc;
        if (int rc = flush_host_locked(src)) return rc;
        CU(cudaStreamSynchronize(src->stream));
    }
    std::lock_guard<std::mutex> lk(dst->mu);
    if (int rc = use_device(dst)) return rc;
    if (int rc = flush_host_locked(dst)) return rc;
    dst->mutation_seq++;
    if (src->device != dst->device) {
        int can = 0;
        CU(cudaDeviceCanAccessPeer(&can, dst->device, src->device));
        if (!can) return fail(DHSA_ECONFIG, "device %d cannot map device %d", dst->device, src->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        (void)cudaGetLastError();
    }
    const void *peers[1] = {src->bits};
    return merge_range_locked(dst, peers, 1, 0, dst->alloc_bytes);
}

extern "C" int dhsa_or_merge_peers(dhsa_sketch_t *dst, const void *const *peer_bits_dev, int n_peers, uint64_t byte_lo,
                                   uint64_t byte_hi)
{
    NEED(dst);
    NEED(peer_bits_dev);
    std::lock_guard<std::mutex> lk(dst->mu);
    if (int rc = use_device(dst)) return rc;
    if (int rc = flush_host_locked(dst)) return rc;
    dst->mutation_seq++;
    return merge_range_locked(dst, peer_bits_dev, n_peers, byte_lo, byte_hi);
}

extern "C" int dhsa_copy_slice_from_peer(dhsa_sketch_t *dst, const void *peer_bits_dev, uint64_t byte_lo,
                                         uint64_t byte_hi)
{
    NEED(dst);
    NEED(peer_bits_dev);
    if ((byte_lo | byte_hi) & 15u) return fail(DHSA_ECONFIG, "slice range must be 16-byte aligned");
    if (byte_lo > byte_hi || byte_hi > dst->alloc_bytes) return fail(DHSA_ECONFIG, "slice range out of bounds");
    if (byte_lo == byte_hi) return DHSA_OK;
    std::lock_guard<std::mutex> lk(dst->mu);
    if (int rc = use_device(dst)) return rc;
    if (int rc = flush_host_locked(dst)) return rc;
    dst->mutation_seq++;
    const uint64_t lo = byte_lo / 16, hi = byte_hi / 16;
    const int grid = grid_for(dst, hi - lo, 256, 8);
    k_copy_slice<<<grid, 256, 0, dst->stream>>>(reinterpret_cast<uint4 *>(dst->bits),
                                               reinterpret_cast<const uint4 *>(peer_bits_dev), lo, hi);
    dst->launches++;
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_or_merge_buffer(dhsa_sketch_t *dst, const void *bits_dev, uint64_t nbytes)
{
    NEED(dst);
    NEED(bits_dev);
    if (nbytes != dst->nbytes) return fail(DHSA_EDATA, "buffer is %llu bytes, sketch holds %llu",
                                           (unsigned long long)nbytes, (unsigned long long)dst->nbytes);
    if ((uintptr_t)bits_dev & 15u) return fail(DHSA_ECONFIG, "buffer must be 16-byte aligned");
    std::lock_guard<std::mutex> lk(dst->mu);
    if (int rc = use_device(dst)) return rc;
    if (int rc = flush_host_locked(dst)) return rc;
    dst->mutation_seq++;
    const void *peers[1] = {bits_dev};
    // whole 16-byte vectors, then the (at most 15-byte) tail of odd-sized toy sketches byte-wise via a padded view:
    // the allocation is padded and zero beyond nbytes on both sides only when the source is itself padded, so
    // merge the aligned prefix here and let the caller pad odd-sized buffers (all real configurations are multiples of 16)
    const uint64_t aligned = nbytes & ~15ull;
    if (aligned != nbytes) return fail(DHSA_ECONFIG, "sketch size %llu is not a multiple of 16 bytes", (unsigned long long)nbytes);
    return merge_range_locked(dst, peers, 1, 0, aligned);
}

// ---- partitioned read-out (multi-GPU) -----------------------------------------------------------
// After the OR reduce-scatter rank q holds the merged byte range q.  Instead of all-gathering the
// merged bits (10 MiB per sketch), each rank counts the zeros of its own range, the counts are
// gathered (4 bytes per cell), and the few cells the candidates' re-estimation needs are read from
// their owners through the peer-mapped pointers.

extern "C" int dhsa_zero_counts_offset(const dhsa_sketch_t *s, uint64_t *byte_offset)
{
    NEED(s);
    NEED(byte_offset);
    *byte_offset = s->alloc_bytes + kCounterBytes;  // from the sketch's base pointer (dhsa_bits_device_ptr / dhsa_ipc_open)
    return DHSA_OK;
}

static int cell_range_of(const dhsa_sketch *s, uint64_t byte_lo, uint64_t byte_hi, uint64_t *cell_lo, uint64_t *cell_hi)
{
    const uint64_t bpe = (uint64_t)s->params.g / 8;
    if (byte_lo > byte_hi || byte_hi > s->alloc_bytes) return fail(DHSA_ECONFIG, "cell range out of bounds");
    if (byte_hi > s->nbytes) byte_hi = s->nbytes;  // the padding of the last range holds no cell
    if (byte_lo > byte_hi) byte_lo = byte_hi;
    if (byte_lo % bpe || byte_hi % bpe)
        return fail(DHSA_ECONFIG, "cell range [%llu, %llu) does not fall on %llu-byte cell boundaries",
                    (unsigned long long)byte_lo, (unsigned long long)byte_hi, (unsigned long long)bpe);
    *cell_lo = byte_lo / bpe, *cell_hi = byte_hi / bpe;
    return DHSA_OK;
}

extern "C" int dhsa_zero_counts_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t byte_hi)
{
    NEED(s);
    uint64_t lo, hi;
    if (int rc = cell_range_of(s, byte_lo, byte_hi, &lo, &hi)) return rc;
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    if (int rc = flush_host_locked(s)) return rc;
    return launch_zero_counts(s, lo, hi);
}

extern "C" int dhsa_gather_zero_counts_from_peer(dhsa_sketch_t *s, const void *peer_bits_dev, uint64_t byte_lo,
                                                 uint64_t byte_hi)
{
    NEED(s);
    NEED(peer_bits_dev);
    uint64_t lo, hi;
    if (int rc = cell_range_of(s, byte_lo, byte_hi, &lo, &hi)) return rc;
    if (lo == hi) return DHSA_OK;
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = use_device(s)) return rc;
    if (int rc = refuse_if_restore_pending(s)) return rc;
    const uint32_t *src = reinterpret_cast<const uint32_t *>(static_cast<const uint8_t *>(peer_bits_dev) + s->alloc_bytes +
                                                             kCounterBytes);
    k_copy_words<<<grid_for(s, hi - lo, 256, 8), 256, 0, s->stream>>>(reinterpret_cast<uint32_t *>(s->zc), src, lo, hi);
    s->launches++;
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_set_cell_owners(dhsa_sketch_t *s, const void *const *bits_dev, const uint64_t *byte_cuts, int n_owners)
{
    NEED(s);
    if (n_owners < 0 || n_owners > DHSA_MAX_OWNERS)
        return fail(DHSA_ECONFIG, "owner count must be 0..%d (got %d)", DHSA_MAX_OWNERS, n_owners);
    CellOwners own;
    memset(&own, 0, sizeof own);
    if (n_owners > 0) {
        NEED(bits_dev);
        NEED(byte_cuts);
        const uint64_t bpe = (uint64_t)s->params.g / 8;
        if (byte_cuts[0] != 0 || byte_cuts[n_owners] < s->nbytes)
            return fail(DHSA_ECONFIG, "owner ranges must cover the sketch: [%llu, %llu) of %llu bytes",
                        (unsigned long long)byte_cuts[0], (unsigned long long)byte_cuts[n_owners],
                        (unsigned long long)s->nbytes);
        for (int q = 0; q < n_owners; q++) {
            if (!bits_dev[q]) return fail(DHSA_ECONFIG, "owner %d has no sketch pointer", q);
            if (byte_cuts[q] > byte_cuts[q + 1] || (byte_cuts[q + 1] < s->nbytes && byte_cuts[q + 1] % bpe))
                return fail(DHSA_ECONFIG, "owner cut %llu is not an ascending %llu-byte cell boundary",
                            (unsigned long long)byte_cuts[q + 1], (unsigned long long)bpe);
            own.base[q] = static_cast<const uint8_t *>(bits_dev[q]);
            own.cut[q] = byte_cuts[q];
        }
        own.cut[n_owners] = byte_cuts[n_owners];
        own.n = n_owners;
    }
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc = refuse_if_restore_pending(s)) return rc;
    s->owners = own;
    s->owners_seq++;
    return DHSA_OK;
}

extern "C" int dhsa_ipc_export(dhsa_sketch_t *s, uint8_t handle_out[64])
{
    NEED(s);
    NEED(handle_out);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    if (int rc = use_device(s)) return rc;
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, s->bits));
    memcpy(handle_out, &h, 64);
    return DHSA_OK;
}

extern "C" int dhsa_ipc_open(int device, const uint8_t handle[64], void **bits_dev)
{
    NEED(handle);
    NEED(bits_dev);
    CU(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    CU(cudaIpcOpenMemHandle(bits_dev, h, cudaIpcMemLazyEnablePeerAccess));
    return DHSA_OK;
}

extern "C" int dhsa_ipc_close(int device, void *bits_dev)
{
    NEED(bits_dev);
    CU(cudaSetDevice(device));
    CU(cudaIpcCloseMemHandle(bits_dev));
    return DHSA_OK;
}

// ------------------------------------------------------------ exact oracle --

struct dhsa_exact {
    int device;
    int sm_count;
    ExactTables t;
    uint64_t pair_cap, host_cap;
    unsigned long long *out;      // collected (host << 32 | count) rows, padded to a power of two
    uint64_t out_cap;
    unsigned long long *n_out;    // device counter
};

static uint64_t pow2_ge(uint64_t v)
{
    uint64_t l = 1;
    while (l < v) l <<= 1;
    return l;
}

extern "C" int dhsa_exact_create(int device, uint64_t expected_pairs, dhsa_exact_t **out)
{
    NEED(out);
    *out = nullptr;
    CU(cudaSetDevice(device));
    dhsa_exact *e = new (std::nothrow) dhsa_exact();
    if (!e) return fail(-1, "out of host memory");
    e->device = device;
    CU(cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, device));
    e->pair_cap = pow2_ge(2 * (expected_pairs < 1024 ? 1024 : expected_pairs));  // load factor <= 0.5
    e->host_cap = e->pair_cap;
    cudaError_t err = cudaMalloc(&e->t.pairs, e->pair_cap * 8);
    if (err == cudaSuccess) err = cudaMalloc(&e->t.hosts, e->host_cap * 8);
    if (err == cudaSuccess) err = cudaMalloc(&e->t.header, 8 * 8);
    if (err == cudaSuccess) err = cudaMalloc(&e->n_out, 8);
    if (err == cudaSuccess) err = cudaMemset(e->t.pairs, 0, e->pair_cap * 8);
    if (err == cudaSuccess) err = cudaMemset(e->t.hosts, 0, e->host_cap * 8);
    if (err == cudaSuccess) err = cudaMemset(e->t.header, 0, 8 * 8);
    if (err != cudaSuccess) {
        cudaFree(e->t.pairs), cudaFree(e->t.hosts), cudaFree(e->t.header), cudaFree(e->n_out);
        delete e;
        return cuda_fail(err, "exact oracle tables");
    }
    e->t.pair_mask = e->pair_cap - 1;
    e->t.host_mask = e->host_cap - 1;
    *out = e;
    return DHSA_OK;
}

extern "C" int dhsa_exact_destroy(dhsa_exact_t *e)
{
    if (!e) return DHSA_OK;
    cudaSetDevice(e->device);
    cudaDeviceSynchronize();
    cudaFree(e->t.pairs), cudaFree(e->t.hosts), cudaFree(e->t.header), cudaFree(e->n_out), cudaFree(e->out);
    delete e;
    return DHSA_OK;
}

static int exact_grid(const dhsa_exact *e, uint64_t nvec)
{
    uint64_t want = (nvec + 255) / 256, cap = (uint64_t)e->sm_count * 8;
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

extern "C" int dhsa_exact_add_pairs(dhsa_exact_t *e, const uint32_t *cand_dev, const uint32_t *opp_dev, uint64_t n,
                                    void *cuda_stream)
{
    NEED(e);
    if (n == 0) return DHSA_OK;
    NEED(cand_dev);
    NEED(opp_dev);
    if (((uintptr_t)cand_dev | (uintptr_t)opp_dev) & 15u || (n & 3u))
        return fail(DHSA_ECONFIG, "exact oracle input must be 16-byte aligned arrays of a multiple of 4 pairs");
    CU(cudaSetDevice(e->device));
    SoaSource src;
    src.cand4 = reinterpret_cast<const uint4 *>(cand_dev);
    src.opp4 = reinterpret_cast<const uint4 *>(opp_dev);
    src.nvec = n / 4;
    k_exact_insert<SoaSource><<<exact_grid(e, src.nvec), 256, 0, (cudaStream_t)cuda_stream>>>(src, e->t);
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_exact_add_records(dhsa_exact_t *e, const void *records_dev, uint64_t n_in_buffer, uint64_t rec_lo,
                                      uint64_t rec_hi, uint32_t window_seconds, uint32_t window_id, int direction,
                                      void *cuda_stream)
{
    NEED(e);
    if (rec_lo >= rec_hi) return DHSA_OK;
    NEED(records_dev);
    if (rec_hi > n_in_buffer) return fail(DHSA_EDATA, "record range exceeds the buffer");
    if (direction < 0 || direction > 2) return fail(DHSA_ECONFIG, "direction must be 0 (src), 1 (dst) or 2 (both)");
    if (((uintptr_t)records_dev & 15u) || (n_in_buffer & 3u))
        return fail(DHSA_ECONFIG, "exact oracle record buffers must be 16-byte aligned and hold a multiple of 4 records");
    CU(cudaSetDevice(e->device));
    for (int pass = 0; pass < 2; pass++) {
        if ((pass == 0 && direction == 1) || (pass == 1 && direction == 0)) continue;
        RecordSource src;
        const uint64_t q_lo = rec_lo / 4, q_hi = (rec_hi + 3) / 4;
        src.rec4 = reinterpret_cast<const uint4 *>(records_dev) + 3 * q_lo;
        src.nquads = q_hi - q_lo;
        src.first_rec = 4 * q_lo;
        src.rec_lo = rec_lo, src.rec_hi = rec_hi;
        src.set_window(window_seconds, window_id);
        src.cand_is_dst = pass;
        src.tally = nullptr, src.tally_late = 0;
        k_exact_insert<RecordSource><<<exact_grid(e, src.nquads), 256, 0, (cudaStream_t)cuda_stream>>>(src, e->t);
    }
    CU(cudaGetLastError());
    return DHSA_OK;
}

extern "C" int dhsa_exact_result(dhsa_exact_t *e, uint64_t min_count, uint64_t *hosts_host, uint64_t *counts_host,
                                 uint64_t cap, uint64_t *n_out, uint64_t *distinct_pairs, uint64_t *distinct_hosts,
                                 void *cuda_stream)
{
    NEED(e);
    NEED(n_out);
    *n_out = 0;
    CU(cudaSetDevice(e->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    unsigned long long header[8];
    CU(cudaMemcpyAsync(header, e->t.header, sizeof header, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (header[2]) return fail(DHSA_ECAPACITY, "exact oracle tables are full (%llu slots); create a larger one",
                               (unsigned long long)e->pair_cap);
    if (distinct_pairs) *distinct_pairs = header[0];
    if (distinct_hosts) *distinct_hosts = header[1];
    const uint64_t want = pow2_ge(header[1] + 1);
    if (want > e->out_cap) {
        cudaFree(e->out);
        e->out = nullptr, e->out_cap = 0;
        CU(cudaMalloc(&e->out, want * 8));
        e->out_cap = want;
    }
    CU(cudaMemsetAsync(e->n_out, 0, 8, st));
    k_exact_collect<<<exact_grid(e, e->host_cap), 256, 0, st>>>(e->t, min_count, e->out, e->out_cap, e->n_out);
    unsigned long long n = 0;
    CU(cudaMemcpyAsync(&n, e->n_out, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    *n_out = n;
    if (n == 0) return DHSA_OK;
    if (n > cap) return fail(DHSA_EDATA, "%llu hosts exceed the output capacity %llu", n, (unsigned long long)cap);
    NEED(hosts_host);
    NEED(counts_host);
    // ascending by host: the packed rows sort as integers
    if (n <= DHSA_SORT_SMEM_MAX) {
        CU(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                DHSA_SORT_SMEM_MAX * (int)sizeof(uint64_t)));
        k_sort_small<<<1, 1024, DHSA_SORT_SMEM_MAX * sizeof(uint64_t), st>>>(
            reinterpret_cast<uint64_t *>(e->out), e->n_out, nullptr, nullptr, 0, nullptr, nullptr);
    } else {
        const uint64_t len = pow2_ge(n);
        const int grid = exact_grid(e, len);
        k_sort_pad<<<grid, 256, 0, st>>>(reinterpret_cast<uint64_t *>(e->out), n, len);
        for (uint64_t kk = 2; kk <= len; kk <<= 1)
            for (uint64_t j = kk >> 1; j > 0; j >>= 1)
                k_bitonic_pass<<<grid, 256, 0, st>>>(reinterpret_cast<uint64_t *>(e->out), len, kk, j);
    }
    CU(cudaGetLastError());
    unsigned long long *rows = (unsigned long long *)malloc(n * 8);
    if (!rows) return fail(-1, "out of host memory");
    cudaError_t err = cudaMemcpyAsync(rows, e->out, n * 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) {
        free(rows);
        return cuda_fail(err, "exact oracle readback");
    }
    for (uint64_t i = 0; i < n; i++) {
        hosts_host[i] = rows[i] >> 32;
        counts_host[i] = rows[i] & 0xFFFFFFFFull;
    }
    free(rows);
    return DHSA_OK;
}

// --------------------------------------------------------- trace generator --

extern "C" int dhsa_generate_trace(int device, const uint32_t *hosts_dev, const uint64_t *prefix_dev,
                                   const uint32_t *bases_dev, uint32_t n_hosts, uint64_t flows, uint64_t dup,
                                   uint64_t seed, uint32_t start_ts, uint32_t window_seconds, uint64_t p_lo,
                                   uint64_t p_hi, void *records_out_dev, uint32_t *cand_out_dev,
                                   uint32_t *opp_out_dev, void *cuda_stream)
{
    if (p_lo >= p_hi) return DHSA_OK;
    NEED(hosts_dev);
    NEED(prefix_dev);
    NEED(bases_dev);
    if (n_hosts == 0 || flows == 0 || dup == 0) return fail(DHSA_ECONFIG, "trace population must be non-empty");
    if (window_seconds == 0) return fail(DHSA_ECONFIG, "window_seconds must be positive (got 0)");
    if (flows > (1ull << 62) / dup) return fail(DHSA_ECONFIG, "flows * duplicate_factor must stay below 2^62");
    const uint64_t total = flows * dup;
    if (p_hi > total) return fail(DHSA_EDATA, "positions [%llu, %llu) exceed the trace's %llu packets",
                                  (unsigned long long)p_lo, (unsigned long long)p_hi, (unsigned long long)total);
    CU(cudaSetDevice(device));
    TraceSpec t;
    t.hosts = hosts_dev, t.prefix = prefix_dev, t.bases = bases_dev;
    t.n_hosts = n_hosts, t.flows = flows, t.total = total;
    t.perm_key = seed;
    uint32_t bits = 2;
    while (bits < 64 && (1ull << bits) < total) bits++;
    t.half_bits = (bits + 1) / 2;
    t.start_ts = start_ts, t.window_seconds = window_seconds;
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint64_t want = (p_hi - p_lo + 255) / 256, cap = (uint64_t)sms * 8;
    const int grid = (int)(want < cap ? want : cap);
    k_generate_trace<<<grid, 256, 0, (cudaStream_t)cuda_stream>>>(t, p_lo, p_hi, static_cast<uint32_t *>(records_out_dev),
                                                                 cand_out_dev, opp_out_dev);
    CU(cudaGetLastError());
    return DHSA_OK;
}

// ----------------------------------------------------------------- probes --

extern "C" int dhsa_probe_l2(int device, int kind, uint64_t buffer_bytes, uint64_t ops, double *ops_per_sec)
{
    NEED(ops_per_sec);
    if (kind < 0 || kind > 3)
        return fail(DHSA_ECONFIG, "probe kind must be 0 (atomic OR), 1 (load), 2 (4 loads + 1 atomic OR) or 3 (32-byte load)");
    uint64_t nwords = buffer_bytes / 4;
    if (nwords < 1024 || (nwords & (nwords - 1)) || nwords > (1ull << 32))
        return fail(DHSA_ECONFIG, "probe buffer must be a power-of-two number of words in [1024, 2^32]");
    CU(cudaSetDevice(device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint32_t *buf = nullptr, *sink = nullptr;
    CU(cudaMalloc(&buf, nwords * 4));
    CU(cudaMalloc(&sink, 4));
    CU(cudaMemset(buf, 0, nwords * 4));
    cudaStream_t st;
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    const int grid = sms * 8;
    float best = 1e30f;
    for (int it = 0; it < 4; it++) {  // first pass warms L2 and the instruction cache
        CU(cudaEventRecord(a, st));
        switch (kind) {
        case 0: k_probe_l2<0><<<grid, 256, 0, st>>>(buf, (uint32_t)(nwords - 1), ops, sink); break;
        case 1: k_probe_l2<1><<<grid, 256, 0, st>>>(buf, (uint32_t)(nwords - 1), ops, sink); break;
        case 2: k_probe_l2<2><<<grid, 256, 0, st>>>(buf, (uint32_t)(nwords - 1), ops, sink); break;
        default: k_probe_l2<3><<<grid, 256, 0, st>>>(buf, (uint32_t)(nwords - 1), ops, sink); break;
        }
        CU(cudaEventRecord(b, st));
        CU(cudaStreamSynchronize(st));
        CU(cudaGetLastError());
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, a, b));
        if (it > 0 && ms < best) best = ms;
    }
    *ops_per_sec = (double)ops / ((double)best * 1e-3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    cudaFree(buf);
    cudaFree(sink);
    return DHSA_OK;
}
