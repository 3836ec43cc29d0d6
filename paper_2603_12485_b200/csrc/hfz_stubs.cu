// Temporary: entry points not implemented yet return HFZ_EINVAL with a message.
#include "hfz_common.cuh"
#define NOT_YET(name) hfz_set_error(name ": not implemented yet"); return HFZ_EINVAL;
extern "C" int hfz_feedback_resolve_allgather(hfz_ctx*, void*, const uint8_t*, uint64_t, uint8_t*, uint64_t*, const uint8_t*, uint8_t*, uint32_t, uint32_t, uint8_t*) { NOT_YET("hfz_feedback_resolve_allgather") }
extern "C" int hfz_edge_record_batch(hfz_ctx*, const uint64_t*, const uint32_t*, const uint64_t*, const uint64_t*, const uint32_t*, uint64_t, uint64_t, uint8_t*, uint64_t*) { NOT_YET("hfz_edge_record_batch") }
extern "C" int hfz_host_edge_record_batch(hfz_ctx*, const uint64_t*, const uint16_t*, uint64_t, uint8_t*) { NOT_YET("hfz_host_edge_record_batch") }
extern "C" uint64_t hfz_havoc_max_out(uint64_t in_len) { uint64_t m = in_len + 1024; return m > HFZ_MAX_INPUT_BYTES ? HFZ_MAX_INPUT_BYTES : m; }
extern "C" int hfz_havoc_batch(hfz_ctx*, const uint8_t*, const uint64_t*, uint64_t, uint64_t*, uint8_t*, const uint64_t*, uint64_t*, uint32_t*) { NOT_YET("hfz_havoc_batch") }
extern "C" int hfz_splice_batch(hfz_ctx*, const uint8_t*, const uint64_t*, const uint32_t*, const uint32_t*, uint64_t, uint64_t*, uint8_t*, const uint64_t*, uint64_t*) { NOT_YET("hfz_splice_batch") }
extern "C" uint64_t hfz_deterministic_count(const uint8_t*, uint64_t) { return 0; }
extern "C" int hfz_deterministic_batch(hfz_ctx*, const uint8_t*, uint64_t, const uint8_t*, uint8_t*, uint64_t) { NOT_YET("hfz_deterministic_batch") }
