/*
 * dhsa_b200.h -- C ABI of the B200-native super point detector hot path.
 *
 * One shared library (paper_1803_11449_b200/csrc -> libdhsa_b200.so, sm_100a)
 * exports exactly the entry points below.  They are what the reference's FFI for
 * this path would bind: each one names the reference interface it replaces
 * (paths relative to /root/reference).  Plain pointers and sizes only -- no
 * torch, numpy or C++ types cross this boundary.  The reference-side binding
 * (a ctypes stub that plugs a GPU sketch into dhsa.engine.WindowSession) is shown
 * in INTEGRATION.md.
 *
 * Conventions
 *   - Every function returns int: 0 ok; 2 config error; 3 data error; 4 capacity
 *     error -- the reference CLI's exit-code classes (pkg/src/dhsa/errors.py:1-5,
 *     pkg/src/dhsa/cli.py:26,33-46); negative = -(1000 + cudaError_t).  Nothing
 *     throws.  dhsa_last_error() returns a thread-local message for the last
 *     non-zero return on the calling thread.
 *   - "_host" pointers are ordinary host memory owned by the caller; pinned
 *     (page-locked) memory is detected and DMA'd directly.  "_dev" pointers are
 *     device memory on the sketch's device.  The caller may free its inputs as
 *     soon as a call returns (pkg/src/dhsa/engine.py:78-86 hands in views).
 *   - A sketch is thread-safe: concurrent calls on one handle are serialised and
 *     stream-ordered (the reference updates one sketch from a thread pool,
 *     pkg/src/dhsa/engine.py:81-86).  Read-out calls see every update issued
 *     before them; dhsa_seal() is the barrier (pkg/src/dhsa/engine.py:89-94).
 *   - Bit layout of the sketch is the reference's snapshot layout: arrays in
 *     order, cells in index order, g/8 bytes per cell, bit b of a cell at bit b%8
 *     of byte b/8 (pkg/src/dhsa/estimator.py:3-5, pkg/src/dhsa/dhla.py:64-67).
 */
#ifndef DHSA_B200_H
#define DHSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DHSA_ABI_VERSION 2

#define DHSA_OK 0
#define DHSA_ECONFIG 2   /* ConfigError    pkg/src/dhsa/errors.py:12 */
#define DHSA_EDATA 3     /* DataError      pkg/src/dhsa/errors.py:16 */
#define DHSA_ECAPACITY 4 /* CapacityError  pkg/src/dhsa/errors.py:20 */

/* Scan kernel variants (dhsa_set_scan_mode). */
#define DHSA_SCAN_RED_ONLY 0      /* one atomic OR per (packet, array), unconditionally        */
#define DHSA_SCAN_TEST_RED 1      /* load the word, atomic only if the bit is still clear      */
#define DHSA_SCAN_TEST_AGG_RED 2  /* as 1, and lanes of a warp hitting one word merge first    */
#define DHSA_SCAN_FLOW_CACHE 3    /* as 2 behind an exact L2-resident cache of scanned pairs   */
#define DHSA_SCAN_AUTO 4          /* default: 3, falling back to 1 for the rest of a window whose
                                     flows do not repeat (hit rate projected from the cache's own
                                     counters below ~1/3): decided by the host between launches and
                                     on the device inside one launch of >= 8M packets             */

typedef struct dhsa_sketch dhsa_sketch_t; /* opaque; replaces dhsa.dhla.Dhla, pkg/src/dhsa/dhla.py:57-68 */

/* The validated parameter record, replaces DhgParams (pkg/src/dhsa/dhg.py:59-118).
 * state_* are the post-tag states: state_dh0 = mix64(seed_dh0 ^ 0x9E3779B97F4A7C15),
 * state_h1 = mix64(seed_h1 ^ 0xD1B54A32D192ED03) (dhg.py:29-30,112-118). */
typedef struct {
    int32_t r;
    int32_t g;
    int32_t k;
    int32_t alpha;
    int32_t key_width;
    int32_t reserved;
    uint64_t state_dh0;
    uint64_t state_h1;
} dhsa_params_t;

/* One reported super point, replaces SuperPointReport (pkg/src/dhsa/dhla.py:50-54). */
typedef struct {
    uint64_t host;
    double estimate;
    int32_t saturated;
    int32_t shared_zero_count; /* SZ before the saturation clamp (dhla.py:183) */
} dhsa_report_t;

/* Everything else one read-out produced. */
typedef struct {
    uint64_t n_candidates;     /* verified, distinct keys (dhla.py:213-217)                 */
    uint64_t n_reports;        /* keys with estimate >= theta (dhla.py:190-194)             */
    int32_t fail_stage;        /* 0, or the stage number of the CapacityError text          */
    int32_t flow_saturated;    /* estimator.py:31                                           */
    uint64_t fail_count;       /* survivor count of the failing stage (dhla.py:270-273)     */
    double flow_count;         /* dhla.py:121-128                                           */
    double psi;                /* dhla.py:130-134                                           */
    double denom;              /* g (1 - psi^r), dhla.py:184                                */
    uint64_t hot_counts[64];   /* |HE(i)|, dhla.py:111-119                                  */
    uint64_t stage_counts[64]; /* survivors after stage 1, 2, ... (r - 2 entries)           */
    int64_t zero_totals[64];   /* ZR(i), dhla.py:126                                        */
    int32_t hot_cut;           /* hot <=> zc < g exp(-theta/g) <=> zc <= hot_cut (dhla.py:45-47,116) */
    int32_t sz_cut;            /* reported <=> estimate >= theta <=> max(SZ, 1) <= sz_cut (dhla.py:183-192) */
} dhsa_restore_info_t;

int dhsa_abi_version(void);
const char *dhsa_last_error(void);

/* ---- lifetime ---------------------------------------------------------------- */

/* Dhla(params) -- allocate and zero r * 2^k * g/8 bytes on `device`
 * (pkg/src/dhsa/dhla.py:60-68).  Re-validates the DhgParams rules
 * (pkg/src/dhsa/dhg.py:78-105) -> DHSA_ECONFIG. */
int dhsa_create(const dhsa_params_t *params, int device, dhsa_sketch_t **out);
/* The reference builds one Dhla per window and drops it after the restore (engine.py:63,165-176);
 * creating a device sketch, its first read-out and freeing it cost tens of milliseconds, so
 * dhsa_destroy parks up to two sketches per (device, parameters) -- zeroed, in their initial
 * state -- and dhsa_create hands a parked one out again.  dhsa_release_cached frees whatever is
 * parked (and the page-locked / staging buffers kept for reuse). */
int dhsa_destroy(dhsa_sketch_t *s);
int dhsa_release_cached(void);
/* Dhla.reset (pkg/src/dhsa/dhla.py:97-99). */
int dhsa_reset(dhsa_sketch_t *s);
/* Dhla.memory_bytes (pkg/src/dhsa/dhla.py:74-76). */
int dhsa_sketch_bytes(const dhsa_sketch_t *s, uint64_t *nbytes);
/* Device address of the bit array (for peers, snapshots, torch views). */
int dhsa_bits_device_ptr(dhsa_sketch_t *s, void **bits_dev);
/* Launch stream.  A new sketch launches on a private non-blocking stream;
 * dhsa_set_stream switches to the caller's cudaStream_t (0 is CUDA's legacy default
 * stream, as torch's default stream reports it), dhsa_set_own_stream switches back.
 * Work queued on the old stream is ordered before work on the new one. */
int dhsa_set_stream(dhsa_sketch_t *s, void *cuda_stream);
int dhsa_set_own_stream(dhsa_sketch_t *s);
int dhsa_get_stream(dhsa_sketch_t *s, void **cuda_stream);
int dhsa_set_scan_mode(dhsa_sketch_t *s, int mode);
/* The kernel variant (0..3) the last vectorised scan launch on this handle used: what
 * DHSA_SCAN_AUTO resolved to. */
int dhsa_scan_mode_used(const dhsa_sketch_t *s, int *mode);
/* Flow cache of DHSA_SCAN_FLOW_CACHE: sets of 8 keys x 4 bytes = 32 bytes.  n_sets is rounded
 * down to a power of two and up to 2g (default 2^20 -> 32 MiB, allocated on first use;
 * 1024 <= n_sets <= 2^27).  The cache only ever skips a packet whose exact key (cand, h1(opp))
 * -- all its bits depend on -- was already scanned into this sketch since its last reset, so
 * the bits are identical with or without it.  stats: keys looked up / found since the reset. */
int dhsa_set_flow_cache(dhsa_sketch_t *s, uint64_t n_sets);
int dhsa_flow_cache_stats(dhsa_sketch_t *s, uint64_t *lookups, uint64_t *hits);
/* Kernel launches issued through this handle so far (bench.py's gpu_launches). */
int dhsa_launch_count(const dhsa_sketch_t *s, uint64_t *n);

/* ---- scan: Backend.update_batch / Dhla.update_batch ------------------------------
 * (pkg/src/dhsa/_core.pyx:52-86, pkg/src/dhsa/_pykernels.py:29-55,
 *  pkg/src/dhsa/dhla.py:87-95).  For every t < n set bit h1(opp[t]) in cell
 *  (i, idx_i(cand[t])) of every array i. */
int dhsa_update_device(dhsa_sketch_t *s, const uint32_t *cand_dev, const uint32_t *opp_dev,
                       uint64_t n);
/* Host arrays.  Small batches -- the reference engine hands over 65,536 pairs at a time from a
 * thread pool (pkg/src/dhsa/engine.py:22,78-86) -- are appended to page-locked accumulation slots
 * by the calling threads, in parallel, and a slot is copied to the device and scanned when it is
 * full or at the next barrier or read-out: the call returns once the caller's arrays have been
 * read, every later read-out sees the batch.  Large page-locked arrays are DMA'd in place. */
int dhsa_update_host(dhsa_sketch_t *s, const uint32_t *cand_host, const uint32_t *opp_host,
                     uint64_t n);
/* dhsa_update_device for arrays produced on another stream than the sketch's (the caller's torch
 * stream, say): ordered after what producer_stream has queued so far; producer_stream in turn
 * waits for the scan, so the arrays may be released to it right after the call.  The sketch
 * keeps its own launch stream. */
int dhsa_update_device_from(dhsa_sketch_t *s, const uint32_t *cand_dev, const uint32_t *opp_dev,
                            uint64_t n, void *producer_stream);
/* WindowSession.seal's barrier (pkg/src/dhsa/engine.py:89-94): drain the stream. */
int dhsa_seal(dhsa_sketch_t *s);

/* ---- the `bits` attribute (pkg/src/dhsa/dhla.py:64-67; written directly by
 *      pkg/src/dhsa/dhla.py:372 and pkg/tests/test_dhla.py:88-90) ----------------- */
int dhsa_download_bits(dhsa_sketch_t *s, uint8_t *bits_host, uint64_t nbytes);
int dhsa_upload_bits(dhsa_sketch_t *s, const uint8_t *bits_host, uint64_t nbytes);
/* The same for a byte range of the array: write_snapshot / read_snapshot (pkg/src/dhsa/dhla.py:321-373)
 * stream the payload between the device and the file in pieces. */
int dhsa_download_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t nbytes, uint8_t *dst_host);
int dhsa_upload_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t nbytes, const uint8_t *src_host);
/* Dhla.estimator(i, j) (pkg/src/dhsa/dhla.py:107-109): the g/8 bytes of one cell (a copy). */
int dhsa_download_cell(dhsa_sketch_t *s, int32_t array, uint64_t index, uint8_t *cell_host,
                       uint64_t nbytes);

/* ---- read-out ---------------------------------------------------------------- */

/* Backend.zero_counts / Dhla.zero_counts (pkg/src/dhsa/_core.pyx:89-118,
 * pkg/src/dhsa/dhla.py:103-105): zc_host = int64 (r, 2^k); zr_host (optional) =
 * per-array totals ZR(i) (pkg/src/dhsa/dhla.py:126). */
int dhsa_zero_counts(dhsa_sketch_t *s, int64_t *zc_host, int64_t *zr_host);
/* The zero_counts= argument of Dhla.hot_sets / estimate_flow_count / _candidate_hosts
 * (pkg/src/dhsa/dhla.py:111-128,198-207): the next one of dhsa_hot_sets / dhsa_estimate /
 * dhsa_candidate_hosts on this handle starts from zc_host (int64 (r, 2^k), each in [0, g])
 * instead of counting the bits. */
int dhsa_use_zero_counts(dhsa_sketch_t *s, const int64_t *zc_host);
/* Dhla.hot_sets (pkg/src/dhsa/dhla.py:111-119, hot_threshold :45-47): row i of
 * lists_host (r x 2^k u64) holds counts_host[i] ascending indices. */
int dhsa_hot_sets(dhsa_sketch_t *s, double theta, uint64_t *lists_host, uint64_t *counts_host);
/* Dhla.estimate_flow_count + bit_set_probability (pkg/src/dhsa/dhla.py:121-134) with the
 * hot-set sizes for `theta`: fills zero_totals, hot_counts, flow_count, flow_saturated,
 * psi and denom of *info. */
int dhsa_estimate(dhsa_sketch_t *s, double theta, dhsa_restore_info_t *info);
/* Dhla._candidate_hosts (pkg/src/dhsa/dhla.py:198-217 with _stage_first :252-274 and
 * _stage_next :277-299): ascending distinct verified keys.  DHSA_ECAPACITY with
 * info->fail_stage / fail_count when a stage exceeds max_candidates. */
int dhsa_candidate_hosts(dhsa_sketch_t *s, double theta, uint64_t max_candidates,
                         uint64_t *hosts_host, uint64_t hosts_cap, dhsa_restore_info_t *info);
/* Dhla.shared_zero_counts (pkg/src/dhsa/dhla.py:136-143). */
int dhsa_shared_zero_counts(dhsa_sketch_t *s, const uint64_t *hosts_host, uint64_t n,
                            int64_t *sz_host);
/* Dhla.restore_superpoints (pkg/src/dhsa/dhla.py:164-196): reports sorted by
 * (-estimate, host).  reports_host holds reports_cap entries; info->n_reports is
 * the true count (DHSA_EDATA if it exceeds reports_cap). */
int dhsa_restore(dhsa_sketch_t *s, double theta, uint64_t max_candidates,
                 dhsa_report_t *reports_host, uint64_t reports_cap, dhsa_restore_info_t *info);
/* The same read-out in two halves, for callers that keep the GPU busy: _begin enqueues the
 * whole chain and returns at once; the caller may queue the next window's reset and scan on
 * this sketch (stream order keeps them behind the read-out) and then collect the reports with
 * _end, which waits only for the read-out.  WindowSession.restore (pkg/src/dhsa/engine.py:96-103)
 * of window k then overlaps the feed of window k + 1.  One read-out may be pending per sketch;
 * other read-out calls fail with DHSA_ECONFIG until it is collected.  _end with too small a
 * buffer returns DHSA_EDATA and leaves the read-out collectable. */
int dhsa_restore_begin(dhsa_sketch_t *s, double theta, uint64_t max_candidates);
int dhsa_restore_end(dhsa_sketch_t *s, dhsa_report_t *reports_host, uint64_t reports_cap,
                     dhsa_restore_info_t *info);

/* ---- the hash group, forward and inverse (stateless: parameters in, no sketch) ---------------
 * dhg.forward_many (pkg/src/dhsa/dhg.py:203-210): indices_host = (n, r) u64, row t the r estimator
 * indices of keys_host[t].
 * dhg.reconstruct_key / reconstruct_many (pkg/src/dhsa/dhg.py:161-185, 213-233): tuples_host =
 * (n, r) u64 index tuples; keys_host[t] = the rebuilt key (meaningless where rejected, as in the
 * reference), ok_host[t] = 1 iff neighbouring blocks agree on their k - alpha overlapping bits, no
 * bit lies above key_width and dh0(key) reproduces index 0 -- the accept predicate the restore
 * stages apply incrementally. */
int dhsa_forward_many(const dhsa_params_t *params, int device, const uint64_t *keys_host, uint64_t n,
                      uint64_t *indices_host);
int dhsa_reconstruct_many(const dhsa_params_t *params, int device, const uint64_t *tuples_host,
                          uint64_t n, uint64_t *keys_host, uint8_t *ok_host);

/* ---- record streams: the window engine's per-record work, fused into the scan --------
 * Records are the reference's 12-byte IPPR trace records (pkg/src/dhsa/ingest.py:20): u32
 * timestamp little-endian, then src and dst IPv4 as u32 big-endian.
 *
 * dhsa_plan_windows: DetectionEngine._run's windowing (pkg/src/dhsa/engine.py:140-149).  A record
 * arrives during the running maximum of ts // window_seconds over the stream so far (seeded with
 * open_window, -1 = none), so the stream splits into contiguous segments, one per window, at the
 * records where that maximum rises; out_host receives those (position, window id) pairs in
 * position order.  DHSA_EDATA if there are more than cap.
 *
 * dhsa_update_records_device: scan records [rec_lo, rec_hi) of a device buffer holding
 * n_in_buffer records into window `window_id`: records with ts // window_seconds == window_id
 * are fed under the direction policy (split_pairs, pkg/src/dhsa/engine.py:179-194: 0 "src",
 * 1 "dst", 2 "both"), the others are late and only counted (engine.py:148-156).
 * dhsa_record_tally: records fed / dropped since the last dhsa_reset (WindowResult.pairs counts
 * fed pairs, i.e. twice the records under "both"; engine.py:49-54,87). */
typedef struct {
    uint64_t position;
    int64_t window_id;
} dhsa_boundary_t;
int dhsa_plan_windows(dhsa_sketch_t *s, const void *records_dev, uint64_t n_records,
                      uint32_t window_seconds, int64_t open_window, dhsa_boundary_t *out_host,
                      uint32_t cap, uint32_t *n_out);
int dhsa_update_records_device(dhsa_sketch_t *s, const void *records_dev, uint64_t n_in_buffer,
                               uint64_t rec_lo, uint64_t rec_hi, uint32_t window_seconds,
                               uint32_t window_id, int direction);
int dhsa_record_tally(dhsa_sketch_t *s, uint64_t *records_fed, uint64_t *records_dropped);
/* The same two counters as they stood when the last collected read-out (dhsa_restore /
 * dhsa_restore_end) ran: copied back with its reports, so no further synchronisation. */
int dhsa_record_tally_at_restore(dhsa_sketch_t *s, uint64_t *records_fed, uint64_t *records_dropped);

/* ---- exact oracle on the GPU: ingest.exact_oracle (pkg/src/dhsa/ingest.py:159-176) -----------
 * Exact number of distinct opposites per candidate host, by a hash set of whole pairs and
 * per-host counters in HBM.  Evaluation tooling for windows too large for the reference's
 * numpy sort/unique; results are exact, not estimates.
 *   create   tables sized for about expected_pairs distinct pairs (grows by re-creation:
 *            DHSA_ECAPACITY from add_* / result means "full, create a larger one")
 *   add_*    insert pairs (device arrays) or raw IPPR records [rec_lo, rec_hi) of window
 *            `window_id` under a direction policy, as dhsa_update_records_device selects them
 *            (window_seconds 0 = no windowing: every record of the range)
 *   result   hosts with count >= min_count, ascending by host */
typedef struct dhsa_exact dhsa_exact_t;
int dhsa_exact_create(int device, uint64_t expected_pairs, dhsa_exact_t **out);
int dhsa_exact_destroy(dhsa_exact_t *e);
int dhsa_exact_add_pairs(dhsa_exact_t *e, const uint32_t *cand_dev, const uint32_t *opp_dev, uint64_t n,
                         void *cuda_stream);
int dhsa_exact_add_records(dhsa_exact_t *e, const void *records_dev, uint64_t n_in_buffer,
                           uint64_t rec_lo, uint64_t rec_hi, uint32_t window_seconds,
                           uint32_t window_id, int direction, void *cuda_stream);
int dhsa_exact_result(dhsa_exact_t *e, uint64_t min_count, uint64_t *hosts_host,
                      uint64_t *counts_host, uint64_t cap, uint64_t *n_out,
                      uint64_t *distinct_pairs, uint64_t *distinct_hosts, void *cuda_stream);

/* ---- synthetic trace generator on the device: ingest.generate_trace's per-record half
 * (pkg/src/dhsa/ingest.py:128-151).  hosts / prefix / bases describe the flow population
 * (n_hosts distinct addresses, exclusive prefix sums of their cardinalities with
 * prefix[n_hosts] = flows, first destination of each host's ramp); the call writes output
 * positions [p_lo, p_hi) of the shuffled, time-ordered stream of flows * dup packets as 12-byte
 * IPPR records and/or (cand, opp) uint32 arrays (null = not wanted).  A rank of a multi-GPU
 * window generates only its own slice. */
int dhsa_generate_trace(int device, const uint32_t *hosts_dev, const uint64_t *prefix_dev,
                        const uint32_t *bases_dev, uint32_t n_hosts, uint64_t flows, uint64_t dup,
                        uint64_t seed, uint32_t start_ts, uint32_t window_seconds, uint64_t p_lo,
                        uint64_t p_hi, void *records_out_dev, uint32_t *cand_out_dev,
                        uint32_t *opp_out_dev, void *cuda_stream);

/* Host -> device staging copy on a caller-chosen stream (cudaMemcpyAsync): DMA straight from
 * page-locked host memory, the driver's bounce buffers otherwise.  Lets the Python engine
 * stage numpy record buffers without routing them through another library. */
int dhsa_copy_to_device_async(int device, void *dst_dev, const void *src_host, uint64_t nbytes,
                              void *cuda_stream);

/* ---- merge: dhsa.dhla.merge (pkg/src/dhsa/dhla.py:305-318) ------------------------ */

/* dst |= src; both handles in this process (same or peer device).  Parameter
 * mismatch -> DHSA_ECONFIG (pkg/src/dhsa/dhla.py:312-315). */
int dhsa_or_merge(dhsa_sketch_t *dst, dhsa_sketch_t *src);
/* dst[byte_lo:byte_hi) |= each peer_bits_dev[p][byte_lo:byte_hi) -- the
 * reduce-scatter-with-OR step of the multi-GPU merge, reading peers over
 * NVLink (peer or IPC-mapped pointers).  byte_lo / byte_hi are multiples of 16. */
int dhsa_or_merge_peers(dhsa_sketch_t *dst, const void *const *peer_bits_dev, int n_peers,
                        uint64_t byte_lo, uint64_t byte_hi);
/* dst[byte_lo:byte_hi) = peer_bits_dev[byte_lo:byte_hi) -- the all-gather step. */
int dhsa_copy_slice_from_peer(dhsa_sketch_t *dst, const void *peer_bits_dev, uint64_t byte_lo,
                              uint64_t byte_hi);
/* dst |= bits_dev (a whole sketch image already on this device, e.g. one slot of an
 * NCCL all-gather buffer). */
int dhsa_or_merge_buffer(dhsa_sketch_t *dst, const void *bits_dev, uint64_t nbytes);
/* Partitioned read-out (BASELINE.json north star: "estimation and restore are partitioned by cell range";
 * SURVEY.md section 8e "K2 over the GPU's own cell range").  After dhsa_or_merge_peers rank q holds the
 * merged byte range q.  Instead of all-gathering the merged bits, each rank counts the zeros of ITS range
 * (the per-range half of Backend.zero_counts, pkg/src/dhsa/_core.pyx:89-118), the counts are gathered
 * (4 bytes per cell instead of g/8), and the cells a candidate's re-estimation ANDs together
 * (shared_zero_counts, pkg/src/dhsa/dhla.py:136-143) are read from their owners through the peer-mapped
 * sketch pointers.  Ranges are byte ranges of the sketch on cell boundaries (multiples of g/8).
 *   dhsa_zero_counts_range             zero counts of the cells in [byte_lo, byte_hi) into the sketch's
 *                                      device-side counts (stream-ordered; the other cells are left alone)
 *   dhsa_zero_counts_offset            where those counts live, as a byte offset from the sketch's base
 *                                      pointer: they share the allocation -- and the IPC handle -- of the bits
 *   dhsa_gather_zero_counts_from_peer  counts of the cells in [byte_lo, byte_hi) copied from a peer's sketch
 *   dhsa_set_cell_owners               n_owners > 0: until it is called again with 0, every read-out call on
 *                                      this handle (restore, candidate hosts, hot sets, shared zero counts)
 *                                      takes the zero counts as gathered and reads cells [byte_cuts[q],
 *                                      byte_cuts[q+1]) from bits_dev[q] (this rank's own base pointer for its
 *                                      own range).  dhsa_download_bits still returns the local array only. */
int dhsa_zero_counts_range(dhsa_sketch_t *s, uint64_t byte_lo, uint64_t byte_hi);
int dhsa_zero_counts_offset(const dhsa_sketch_t *s, uint64_t *byte_offset);
int dhsa_gather_zero_counts_from_peer(dhsa_sketch_t *s, const void *peer_bits_dev, uint64_t byte_lo,
                                      uint64_t byte_hi);
int dhsa_set_cell_owners(dhsa_sketch_t *s, const void *const *bits_dev, const uint64_t *byte_cuts,
                         int n_owners);
/* CUDA IPC plumbing so one-process-per-GPU ranks can map each other's bit arrays. */
int dhsa_ipc_export(dhsa_sketch_t *s, uint8_t handle_out[64]);
int dhsa_ipc_open(int device, const uint8_t handle[64], void **bits_dev);
int dhsa_ipc_close(int device, void *bits_dev);

/* Host-only self test of the helper-thread copy pool behind dhsa_update_host (no CUDA call, runs
 * without a GPU): `threads` concurrent callers x `iterations` two-array copies of random sizes up to
 * bytes_each, each verified; *mismatches = copies that differed from their source. */
int dhsa_selftest_copy_pool(uint64_t bytes_each, int iterations, int threads, uint64_t *mismatches);

/* ---- measurement -------------------------------------------------------------
 * Random-address L2 probe used for the scan roofline: `ops` 32-bit operations at
 * hashed word addresses inside a `buffer_bytes` buffer.  kind 0 = atomic OR
 * (RED), 1 = load, 2 = four loads + one RED per `ops` count of four (do loads and REDs
 * share a limit?), 3 = 256-bit load of a whole 32-byte sector (the flow-cache lookup's
 * shape).  Returns the rate in operations per second. */
int dhsa_probe_l2(int device, int kind, uint64_t buffer_bytes, uint64_t ops, double *ops_per_sec);

#ifdef __cplusplus
}
#endif
#endif /* DHSA_B200_H */
