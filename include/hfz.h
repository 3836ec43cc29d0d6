/*
 * hfz.h -- C-ABI of the B200-native coverage-feedback core ("hetfuzz on B200").
 *
 * This is the drop-in boundary: plain pointers and sizes, int status codes, no
 * exceptions, no torch/C++ types.  The reference has no FFI of its own -- its
 * hot path sits behind the C++ headers proj/include/hetfuzz/{coverage,rng,
 * engine}.hpp (statically linked, proj/CMakeLists.txt:14-23) and the pybind11
 * module proj/python/bindings.cpp:310-350.  Each entry point below names the
 * reference interface it replaces; the headers under include/hetfuzz/ re-create the
 * reference's C++ API on top of these calls and INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *   - every function returns 0 (HFZ_OK) or an HFZ_E* code; hfz_last_error()
 *     gives a thread-local message.  Nothing throws across the ABI.
 *   - all *device* pointers are caller-owned CUDA device memory on the
 *     context's device; the library never frees or reallocates them.  Scratch
 *     (first-occurrence table, per-exec Admit flags, novelty delta) is owned by the
 *     context.
 *   - work is enqueued on the context's stream and is asynchronous unless the
 *     function name ends in _host (those take HOST buffers and synchronise).
 *   - there is NO CPU fallback: without a CUDA device every call fails with
 *     HFZ_ECUDA.
 *
 * Raw map record ("trace_bits" of one execution), S logical slots, H = S/2:
 *     [ H x u8  host counters   (CoverageMap::host_,   coverage.hpp:19) ]
 *     [ H x u32 device counters (CoverageMap::device_, coverage.hpp:20) ]
 *   = 5*H bytes (163,840 B for the reference's S = 65,536).  Records of a batch
 *   are contiguous; the base pointer must be 16-byte aligned.
 * Virgin map: S bytes, REFERENCE polarity (0 = never seen, class bits are OR-ed
 * in; VirginMap, coverage.hpp:155-180).  AFL's AND-merge == bitwise OR here.
 */
#ifndef HFZ_H_
#define HFZ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define HFZ_API
#else
#define HFZ_API __attribute__((visibility("default")))
#endif

#define HFZ_VERSION 120 /* 0.1.2: + packed list ingest, peer buffers over CUDA IPC (0.1.1: sparse / compact lists, peer-memory resolve, serial-stream havoc with host buffers) */

enum {
  HFZ_OK = 0,
  HFZ_EINVAL = 1,   /* bad argument (null pointer, unsupported map size, ...) */
  HFZ_ECUDA = 2,    /* CUDA runtime error; see hfz_last_error() */
  HFZ_ENOMEM = 3,   /* scratch allocation failed */
  HFZ_ECAP = 4,     /* batch exceeds a capacity fixed at context creation */
  HFZ_ENCCL = 5     /* NCCL not loadable / collective failed */
};

/* Admit codes: enum class Admit, coverage.hpp:182-186 */
enum { HFZ_ADMIT_NONE = 0, HFZ_ADMIT_NEW_COUNTS = 1, HFZ_ADMIT_NEW_EDGES = 2 };

#define HFZ_MAX_INPUT_BYTES (1u << 20) /* kMaxInputBytes, engine.hpp:17 */

typedef struct hfz_ctx hfz_ctx;

HFZ_API int hfz_version(void);
HFZ_API const char* hfz_last_error(void);

/*
 * Context: one per (host thread, GPU).  map_slots = S (power of two,
 * 1024 <= S <= 2^24; the reference's kMapSize is 65536, coverage.hpp:13).
 * stream is a cudaStream_t (NULL = the legacy default stream).
 * Threading contract of SPEC.md:124-125 is kept: one writer per virgin map.
 */
HFZ_API int hfz_ctx_create(hfz_ctx** out, int device, uint32_t map_slots, void* stream);
HFZ_API int hfz_ctx_destroy(hfz_ctx* ctx);
HFZ_API int hfz_ctx_set_stream(hfz_ctx* ctx, void* stream);
HFZ_API int hfz_ctx_sync(hfz_ctx* ctx);
HFZ_API uint32_t hfz_ctx_map_slots(const hfz_ctx* ctx);
HFZ_API uint64_t hfz_record_bytes(uint32_t map_slots);
/* Tuning knobs, mostly for bench/profiling: key in {"scan_warps","scan_row","scan_prefetch","virgin_smem","scan_small","time_scan","stage_execs","sparse_chunk","sparse_native","scan_pipe"} */
HFZ_API int hfz_ctx_set_option(hfz_ctx* ctx, const char* key, int64_t value);
/* Kernels launched by this context since creation (for bench.py's gpu_launches). */
HFZ_API uint64_t hfz_ctx_launch_count(const hfz_ctx* ctx);
/* Live kernel timing for the roofline line of bench.py: with option "time_scan" = 1 every
 * launch of the scan kernel (K2, the dominant kernel) is bracketed by CUDA events on the
 * context's stream.  key in {"scan_ms_total", "scan_launches"}; reading synchronises the
 * stream and resets the accumulators. */
HFZ_API int hfz_ctx_get_stat(hfz_ctx* ctx, const char* key, double* out);

/* ------------------------------------------------------------------------- */
/* Fused feedback (K2): replaces, for a whole batch folded IN EXEC ORDER,
 *   classify_trace   coverage.hpp:152, src/coverage.cpp:58-72
 *   trace_signature  coverage.hpp:199, src/coverage.cpp:89-97 (Full and Simple)
 *   has_new_bits     coverage.hpp:191, src/coverage.cpp:74-87 (+VirginMap::observe)
 * i.e. lines 471-478 of Campaign::run_one (src/engine.cpp).
 *
 *   raw_maps          device, n_exec records
 *   virgin_inout      device, S bytes; on return = virgin after the last exec
 *   edge_counts_inout device, 2 x u64 {host_edges, device_edges}
 *                     (VirginMap::host_edges/device_edges, coverage.hpp:163-164)
 *   classed_out       device, n_exec x S bytes or NULL (ClassedTrace::classed)
 *   admit_out         device, n_exec x u8 Admit codes, exactly the sequential ones
 *   sig_full_out / sig_simple_out   device, n_exec x u64
 *   nnz_out           device, n_exec x u32 (ClassedTrace::nonzero.size()) or NULL
 *
 * Context-owned scratch (grown geometrically, kept): 32 x S bytes of first-occurrence table (two of
 * them once a small batch has been folded), 5 bytes per exec of the largest batch seen (Admit flags), and -- for
 * batches of up to 8,192 execs, which are folded by one cooperative launch over ordered slot lists --
 * n_exec x S x 4 bytes of list address space of which only the used prefix of each 4 KB piece's range
 * is ever touched (2 GB at 8,192 execs of 65,536 slots; option "scan_two_stage" = 0 turns that path
 * off, any other value is its batch-size limit).
 */
HFZ_API int hfz_feedback_batch(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                               uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                               uint8_t* classed_out, uint8_t* admit_out,
                               uint64_t* sig_full_out, uint64_t* sig_simple_out,
                               uint32_t* nnz_out);

/* Same call with HOST buffers (pageable or pinned): copies in chunks through
 * context-owned staging, overlapping H2D with the kernels; synchronous. */
HFZ_API int hfz_feedback_batch_host(hfz_ctx* ctx, const uint8_t* raw_maps_host, uint64_t n_exec,
                                    uint8_t* virgin_inout_host, uint64_t* edge_counts_inout_host,
                                    uint8_t* classed_out_host, uint8_t* admit_out_host,
                                    uint64_t* sig_full_out_host, uint64_t* sig_simple_out_host,
                                    uint32_t* nnz_out_host);

/* ------------------------------------------------------------------------- */
/* Sparse ingest: the same fold, fed with per-exec TOUCHED-SLOT LISTS instead of dense records.
 * A raw map is ~2 % dense; the reference's runtime already keeps a dirty-slot list beside its
 * device counters (Runtime::bump_counter / reset_device_coverage, src/hdvm.cpp:356-366) and
 * classify_trace reduces a map to its non-zero list (src/coverage.cpp:58-72).  A list ships
 * ~10 KB per exec over PCIe instead of 163,840 B.
 *
 *   entries    n_total x {u32 slot, u32 count} pairs, 8-byte aligned.  Exec e owns pairs
 *              [entry_off[e], entry_off[e+1]); ANY order inside an exec.  Listing a slot twice
 *              with the SAME count is harmless (it is one slot); with different counts it is
 *              unspecified which one each output uses.  slot < S/2 is a host counter
 *              (count & 0xff is stored, CoverageMap::host_), S/2 <= slot < S a device counter
 *              (full u32, CoverageMap::device_).  count 0 leaves the slot unvisited.  Pairs
 *              with slot >= S are ignored and counted: the _host call then returns HFZ_EINVAL
 *              after completing the fold.
 *   entry_off  (n_exec+1) x u64, non-decreasing absolute indices into `entries` (entry_off[0] need
 *              not be 0: pass entry_off + k to fold execs k.. of a larger batch)
 * Outputs and in/out state exactly as hfz_feedback_batch: results are bit-identical to the
 * dense call on the maps the lists describe.  For S <= 2^20 the lists are folded directly
 * (rank + chain kernels, option "sparse_native" = 1, the default; the device-buffer call reads
 * entry_off[n_exec] back once to size its scratch, i.e. it synchronises the stream before it
 * enqueues); otherwise, or with "sparse_native" = 0, they are expanded chunk by chunk into a
 * context-owned, all-zero staging buffer (option "sparse_chunk" = execs per chunk, default
 * ~1.25 GB of records) which the K2 scan then streams.
 */
HFZ_API int hfz_feedback_batch_sparse(hfz_ctx* ctx, const uint32_t* entries, const uint64_t* entry_off,
                                      uint64_t n_exec, uint8_t* virgin_inout,
                                      uint64_t* edge_counts_inout, uint8_t* classed_out,
                                      uint8_t* admit_out, uint64_t* sig_full_out,
                                      uint64_t* sig_simple_out, uint32_t* nnz_out);
/* HOST buffers (pinned for full PCIe speed, see hfz_host_alloc): the pairs stream in on a copy
 * stream chunk by chunk while earlier chunks are folded; synchronous. */
HFZ_API int hfz_feedback_batch_sparse_host(hfz_ctx* ctx, const uint32_t* entries_host,
                                           const uint64_t* entry_off_host, uint64_t n_exec,
                                           uint8_t* virgin_inout_host, uint64_t* edge_counts_inout_host,
                                           uint8_t* classed_out_host, uint8_t* admit_out_host,
                                           uint64_t* sig_full_out_host, uint64_t* sig_simple_out_host,
                                           uint32_t* nnz_out_host);
/* Compact lists, for maps of at most 65,536 slots: the same touched-slot lists at FOUR bytes per
 * pair.  compact = u32 words `slot | count << 16` for counts below 65,536 (host counters always
 * fit); wide = {u32 slot, u32 count} pairs as above for the larger device counters (wide and
 * wide_off may be NULL when there are none).  Exec e owns compact[compact_off[e] ..
 * compact_off[e+1]) and wide[wide_off[e] .. wide_off[e+1]); a slot belongs in ONE of the two lists.
 * Everything else as hfz_feedback_batch_sparse_host; needs the list-native fold (HFZ_EINVAL when
 * map_slots > 2^20 or option "sparse_native" = 0). */
HFZ_API int hfz_feedback_batch_compact_host(hfz_ctx* ctx, const uint32_t* compact_host,
                                            const uint64_t* compact_off_host, const uint32_t* wide_host,
                                            const uint64_t* wide_off_host, uint64_t n_exec,
                                            uint8_t* virgin_inout_host, uint64_t* edge_counts_inout_host,
                                            uint8_t* classed_out_host, uint8_t* admit_out_host,
                                            uint64_t* sig_full_out_host, uint64_t* sig_simple_out_host,
                                            uint32_t* nnz_out_host);
/* Packed lists, for the reference's map of exactly 65,536 slots (H = 32,768): the same touched-slot lists
 * at THREE bytes per host-half slot and FOUR per device-half slot, no second list for large counters.
 *   host3  bytes; entry i = {slot & 0xff, slot >> 8, count u8} at bytes [3i, 3i + 3), slot < 32,768, count 0 =
 *          ignored.  Exec e owns entries [host3_off[e], host3_off[e+1]); every exec's entry count is padded
 *          with zero entries to a MULTIPLE OF FOUR (offsets are multiples of four; the base is 4-byte
 *          aligned), so four entries are three aligned words on the device.
 *   dev17  u32 words (slot - 32768) | min(count, 65536) << 15: the device ladder's last rung starts at
 *          65,536 (src/coverage.cpp:21-32), so the clip keeps every class; count 0 = ignored.
 *          Exec e owns words [dev17_off[e], dev17_off[e+1]).
 * ~4.1 KB per exec of the bench batch against ~5.0 KB of the compact form: the host call is PCIe-bound, so
 * that is what it gains.  Everything else as hfz_feedback_batch_compact_host. */
HFZ_API int hfz_feedback_batch_packed_host(hfz_ctx* ctx, const uint8_t* host3_host, const uint64_t* host3_off_host,
                                           const uint32_t* dev17_host, const uint64_t* dev17_off_host,
                                           uint64_t n_exec, uint8_t* virgin_inout_host,
                                           uint64_t* edge_counts_inout_host, uint8_t* classed_out_host,
                                           uint8_t* admit_out_host, uint64_t* sig_full_out_host,
                                           uint64_t* sig_simple_out_host, uint32_t* nnz_out_host);
/* The same over SEVERAL packed batches -- one per packing thread of the host, say -- folded in the order given by
 * ONE call: every list is queued on the copy stream up front, batch k + 1 streams in under the fold of batch k,
 * and the call synchronises once.  host3[k] / host3_off[k] / dev17[k] / dev17_off[k] / n_exec[k] describe batch k
 * as above (HOST arrays of n_batches pointers / counts); the outputs hold sum(n_exec) entries in batch order.
 * Classed maps are not returned by this form. */
HFZ_API int hfz_feedback_batch_packed_host_v(hfz_ctx* ctx, uint32_t n_batches, const uint8_t* const* host3_host,
                                             const uint64_t* const* host3_off_host, const uint32_t* const* dev17_host,
                                             const uint64_t* const* dev17_off_host, const uint64_t* n_exec,
                                             uint8_t* virgin_inout_host, uint64_t* edge_counts_inout_host,
                                             uint8_t* admit_out_host, uint64_t* sig_full_out_host,
                                             uint64_t* sig_simple_out_host, uint32_t* nnz_out_host);
/* lists -> dense records (device buffers; raw_maps_out is overwritten, n_exec records) */
HFZ_API int hfz_expand_sparse(hfz_ctx* ctx, const uint32_t* entries, const uint64_t* entry_off,
                              uint64_t n_exec, uint8_t* raw_maps_out);
/* Page-locked host memory for hosts that do not link the CUDA runtime themselves. */
HFZ_API int hfz_host_alloc(void** out, uint64_t bytes);
HFZ_API int hfz_host_free(void* p);

/* The two halves of hfz_feedback_batch, exposed for multi-GPU sharding
 * (SURVEY.md 8e).  Rank r owns a contiguous exec range of the global batch.
 *
 * scan:    one HBM pass over the rank's maps against the batch-start virgin V0:
 *          classed maps, signatures, nnz, and this rank's novelty delta
 *          D_r = OR of class bits not in V0 (S bytes, written to delta_out).
 * resolve: given all ranks' deltas (n_ranks x S bytes, rank-major, e.g. the
 *          output of an NCCL allgather of delta_out), computes the exact
 *          sequential Admit codes of this rank's execs against
 *          P_r = V0 | OR_{q<r} D_q, then folds virgin_inout = V0 | OR_q D_q in
 *          fixed rank order and bumps the edge counters.  Identical on every
 *          rank and identical to the single-rank sequential oracle.
 *          The codes come from the scan's first-occurrence table alone (one
 *          thread per slot): raw_maps is not read again and may be NULL; the
 *          parameter is kept for ABI stability.
 * With n_ranks == 1 and deltas == delta_out the pair equals hfz_feedback_batch.
 */
HFZ_API int hfz_feedback_scan(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                              const uint8_t* virgin_v0, uint8_t* classed_out,
                              uint64_t* sig_full_out, uint64_t* sig_simple_out,
                              uint32_t* nnz_out, uint8_t* delta_out);
HFZ_API int hfz_feedback_resolve(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                 uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                 const uint8_t* deltas, uint32_t n_ranks, uint32_t rank,
                                 uint8_t* admit_out);

/* Peer-memory form of hfz_feedback_resolve: no allgather, no staging copy.  delta_ptrs (HOST
 * array of n_ranks <= 16 device pointers) names every rank's novelty delta where its scan wrote
 * it: own memory for this rank, peer memory mapped into this device's address space for the
 * others (cudaIpcOpenMemHandle, CUDA VMM or torch symmetric memory; NVLink / NVSwitch loads).
 * The merge kernel reads the R x S bytes straight from their owners in fixed rank order.  The
 * caller orders the call after every rank's scan (and the next scan after every rank's resolve)
 * with a device- or host-side barrier. */
HFZ_API int hfz_feedback_resolve_peers(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                       uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                       const uint8_t* const* delta_ptrs, uint32_t n_ranks, uint32_t rank,
                                       uint8_t* admit_out);

/* Buffers for that table when the ranks are separate processes (one per GPU): hfz_peer_alloc makes a
 * device buffer of its own (zero-filled) and exports its CUDA IPC handle; every other rank passes the
 * handle -- exchanged once at start-up by whatever the host uses (torch.distributed, MPI, a socket) -- to
 * hfz_peer_open and gets a pointer valid on ITS device: same device or any device with peer access
 * (NVLink / NVSwitch).  The scan writes its delta into the rank's own buffer (delta_out), the ranks
 * meet at a barrier, and hfz_feedback_resolve_peers reads all of them in place.  Close before the owner frees. */
#define HFZ_PEER_HANDLE_BYTES 64
HFZ_API int hfz_peer_alloc(hfz_ctx* ctx, uint64_t bytes, void** dev_ptr_out, uint8_t* handle_out /* [64] */);
HFZ_API int hfz_peer_open(hfz_ctx* ctx, const uint8_t* handle /* [64] */, void** dev_ptr_out);
HFZ_API int hfz_peer_close(hfz_ctx* ctx, void* dev_ptr);  /* a pointer from hfz_peer_open */
HFZ_API int hfz_peer_free(hfz_ctx* ctx, void* dev_ptr);   /* a pointer from hfz_peer_alloc */

/* K4 alone: virgin_inout |= OR_q deltas[q] in rank order, edge counters updated
 * (bitwise OR in reference polarity == AFL's virgin AND-merge). */
HFZ_API int hfz_virgin_merge(hfz_ctx* ctx, uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                             const uint8_t* deltas, uint32_t n_ranks);

/* allgather + resolve in one call for C/C++ hosts: nccl_comm is an ncclComm_t
 * (libnccl is dlopen()ed on first use; HFZ_ENCCL if unavailable). */
HFZ_API int hfz_feedback_resolve_allgather(hfz_ctx* ctx, void* nccl_comm, const uint8_t* raw_maps,
                                           uint64_t n_exec, uint8_t* virgin_inout,
                                           uint64_t* edge_counts_inout, const uint8_t* delta_local,
                                           uint8_t* deltas_scratch, uint32_t n_ranks,
                                           uint32_t rank, uint8_t* admit_out);

/* ------------------------------------------------------------------------- */
/* Edge record (K1): replaces DeviceThreadCtx::Impl::edge + Runtime::bump_counter
 * (src/hdvm.cpp:415-431, 362-366), the thread/warp enumeration of
 * Runtime::do_launch (src/hdvm.cpp:556-603) and merge_device_into_map
 * (coverage.hpp:204-205) for a batch of executions.
 *
 *   launch_off  device, (n_exec+1) x u64: exec e owns launches [launch_off[e], launch_off[e+1])
 *   dims        device, n_launch x 6 x u32: grid.x,y,z, block.x,y,z  (LaunchConfig, hdvm.hpp:31-45)
 *   thread_off  device, (n_launch+1) x u64: first simulated thread of each launch; threads are
 *               numbered block-linear outer, linear-in-block inner (hdvm.cpp:562,583)
 *   ev_off      device, (n_threads+1) x u64: thread t's sites are sites[ev_off[t], ev_off[t+1])
 *   sites       device, u32 basic-block ids in execution order
 *   raw_maps    device, n_exec records; the DEVICE HALF of each is overwritten with the
 *               saturating warp counters (host half untouched)
 *   warp_events_out device, n_exec x u64 (ExecutionReport::warp_edge_events) or NULL
 *
 * The call reads a few batch sizes back once (it synchronises the stream before its main launches).
 * Context-owned scratch, grown on demand and kept: 4 bytes per trace event of a chunk of execs (the
 * bump lists; option "edge_scratch_mb", default 2048, bounds it by cutting the batch into chunks of
 * whole execs -- one exec larger than the bound still gets what it needs) + 144 bytes per simulated
 * warp of the chunk + 29 bytes per launch / exec of the batch.  Option "edge_flat" = 0 sends every
 * exec through the per-exec kernel (which execs whose launches differ in geometry always take);
 * its only scratch is 4 bytes per simulated thread of the largest launch per SM.
 */
HFZ_API int hfz_edge_record_batch(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                  const uint64_t* thread_off, const uint64_t* ev_off,
                                  const uint32_t* sites, uint64_t n_exec, uint64_t n_launch,
                                  uint8_t* raw_maps, uint64_t* warp_events_out);

/* Edge record straight into touched-slot lists: the device half never has to exist as a dense record
 * between K1 and K2.  As hfz_edge_record_batch, plus per exec a list of (logical slot, count) pairs --
 * the form hfz_feedback_batch_sparse folds (logical slot = map_slots / 2 + device slot: the device half is
 * the upper half of the map, coverage.hpp:13-15,88-91) -- at a fixed stride:
 *   entries_out   device, n_exec x entry_cap x 2 x u32; exec e's pairs are the first n_slots_out[e] of
 *                 [e * entry_cap, (e + 1) * entry_cap), in no particular order, the rest {0, 0} (padding the
 *                 fold ignores), so entry_off[e] = e * entry_cap describes the batch
 *   entry_cap     pairs per exec; the counting kernel's dirty-slot table holds 6,144 distinct slots
 *   n_slots_out   device, n_exec x u32: distinct device slots of the exec, or 0xffffffff when the exec is NOT
 *                 listed (more distinct slots than entry_cap or than the table holds, or launches of differing
 *                 geometry): its list is all padding and the caller takes the dense record for it
 *   raw_maps      as above, or NULL: lists only (nothing dense is written; warp_events_out as above)
 * Needs option "edge_flat" = 1 (the default). */
HFZ_API int hfz_edge_record_batch_lists(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                        const uint64_t* thread_off, const uint64_t* ev_off,
                                        const uint32_t* sites, uint64_t n_exec, uint64_t n_launch,
                                        uint8_t* raw_maps, uint64_t* warp_events_out, uint32_t* entries_out,
                                        uint32_t entry_cap, uint32_t* n_slots_out);

/* Host edge record: host_edge_update + CoverageMap::host_increment
 * (coverage.hpp:24-32,79-84) for batched u16 host site traces.
 *   site_off device (n_exec+1) x u64; sites device u16; fills the HOST HALF. */
HFZ_API int hfz_host_edge_record_batch(hfz_ctx* ctx, const uint64_t* site_off,
                                       const uint16_t* sites, uint64_t n_exec, uint8_t* raw_maps);

/* ------------------------------------------------------------------------- */
/* Batched havoc (K3): replaces havoc_mutant(input, Rng&) (engine.hpp:29-30,
 * src/engine.cpp:119-193), one independent Rng per slot (rng.hpp:11-46).
 *   in_bytes / in_off   device, inputs back to back, (n+1) x u64 offsets
 *   rng_state_inout     device, n x u64 splitmix64 states (Rng(seed) has state == seed);
 *                       on return the state after the slot's draws
 *   out_bytes           device, slot j's output starts at out_off[j]; it must hold
 *                       hfz_havoc_max_out(len_j) bytes
 *   out_off             device, (n+1) x u64 (capacity layout, caller-computed)
 *   out_len             device, n x u64 actual mutant lengths
 *   draws_out           device, n x u32 draws consumed, or NULL
 */
HFZ_API uint64_t hfz_havoc_max_out(uint64_t in_len);
HFZ_API int hfz_havoc_batch(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                            uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                            const uint64_t* out_off, uint64_t* out_len, uint32_t* draws_out);

/* Serial-stream mode: ONE Rng threaded through n mutants in slot order, as
 * Campaign::fuzz_entry does (src/engine.cpp:561-562).  A length-only dry run of every slot on the
 * device yields the state each slot starts from (slot_states_out, feed it to hfz_havoc_batch) and
 * leaves the stream's state after the n-th mutant in stream_state_inout (device, 1 x u64). */
HFZ_API int hfz_havoc_serial_plan(hfz_ctx* ctx, const uint64_t* in_off, uint64_t n,
                                  uint64_t* stream_state_inout, uint64_t* slot_states_out);

/* Serial-stream havoc with HOST buffers: plan + batch in one synchronous call.  The n mutants
 * consume ONE Rng in slot order exactly like the havoc loop of Campaign::fuzz_entry
 * (src/engine.cpp:561-562); *stream_state_inout (host) is the campaign Rng's state. */
HFZ_API int hfz_havoc_serial_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                  uint64_t n, uint64_t* stream_state_inout, uint8_t* out_bytes,
                                  const uint64_t* out_off, uint64_t* out_len);

/* splice_mutant (engine.hpp:33-35, src/engine.cpp:195-204): slot j splices
 * a = input a_idx[j], b = input b_idx[j] of the same packed input set. */
HFZ_API int hfz_splice_batch(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                             const uint32_t* a_idx, const uint32_t* b_idx, uint64_t n,
                             uint64_t* rng_state_inout, uint8_t* out_bytes,
                             const uint64_t* out_off, uint64_t* out_len);

/* deterministic_mutants (engine.hpp:25-26, src/engine.cpp:53-117) of ONE input:
 * count first (host arithmetic), then materialise count x in_len bytes. */
HFZ_API uint64_t hfz_deterministic_count(const uint8_t* in_host, uint64_t in_len);
HFZ_API int hfz_deterministic_batch(hfz_ctx* ctx, const uint8_t* in_dev, uint64_t in_len,
                                    const uint8_t* in_host, uint8_t* out_dev, uint64_t count);

/* HOST-buffer forms of the mutators (what include/hetfuzz/engine.hpp and the pybind-style
 * single-item calls use): same semantics, all pointers are host memory, synchronous. */
HFZ_API int hfz_havoc_batch_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                 uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                                 const uint64_t* out_off, uint64_t* out_len, uint32_t* draws_out);
HFZ_API int hfz_splice_batch_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                  uint64_t n_inputs, const uint32_t* a_idx, const uint32_t* b_idx,
                                  uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                                  const uint64_t* out_off, uint64_t* out_len);
HFZ_API int hfz_deterministic_host(hfz_ctx* ctx, const uint8_t* in, uint64_t in_len, uint8_t* out,
                                   uint64_t count);

/* ------------------------------------------------------------------------- */
/* Signature seen-sets and dispatch flags: the std::set<uint64_t> pair of
 * Campaign (src/engine.cpp:319) with count()-then-insert() semantics in exec order
 * (src/engine.cpp:474-478) and should_sanitize (src/sanitizers.cpp:283-296), on the device.
 * capacity: power of two; a set refuses to grow past 3/4 of it (HFZ_ECAP). */
typedef struct hfz_sigset hfz_sigset;
HFZ_API int hfz_sigset_create(hfz_ctx* ctx, uint64_t capacity, hfz_sigset** out);
HFZ_API int hfz_sigset_destroy(hfz_sigset* set);
HFZ_API int hfz_sigset_size(hfz_sigset* set, uint64_t* size_out); /* synchronises */
/* seen_out[i] = 1 iff sigs[i] was in the set before the call or equals sigs[j], j < i */
HFZ_API int hfz_sigset_seen_insert(hfz_ctx* ctx, hfz_sigset* set, const uint64_t* sigs, uint64_t n,
                                   uint8_t* seen_out);
/* strategy: 0 AllTrace, 1 UniqueTrace, 2 SimpleTrace, 3 CoverageIncrease (sanitizers.hpp:70-75) */
HFZ_API int hfz_dispatch_batch(hfz_ctx* ctx, hfz_sigset* full_set, hfz_sigset* simple_set,
                               const uint64_t* sig_full, const uint64_t* sig_simple,
                               const uint8_t* admit, uint64_t n, int strategy,
                               uint8_t* full_seen_out, uint8_t* simple_seen_out,
                               uint8_t* sanitize_out);

/* Rng helpers (host side, O(1)): rng.hpp:15-21,39-42.  State after k draws =
 * state + k*gamma; split() child seed of the tag-th split from a parent state. */
HFZ_API uint64_t hfz_rng_jump(uint64_t state, uint64_t k);
HFZ_API uint64_t hfz_rng_next(uint64_t* state);
HFZ_API uint64_t hfz_rng_below(uint64_t* state, uint64_t n);
HFZ_API uint64_t hfz_rng_split(uint64_t* state, uint64_t tag);

#ifdef __cplusplus
}
#endif
#endif /* HFZ_H_ */
