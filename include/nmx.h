/* nmx.h -- C ABI of libnmx.so, the B200 (sm_100a) traffic-matrix hot path.
 *
 * The reference (`netmeter`, /root/reference/pkg/src/netmeter) is pure Python
 * + numpy and has no FFI; the Python package paper_2510_14050_b200 binds these
 * entry points with ctypes and re-exposes the reference's own function names.
 * Each entry cites the reference interface it replaces.
 *
 * Conventions
 *   - every function returns an int status: NMX_OK (0) or a negative code;
 *     nmx_last_error() returns the calling thread's message for the last failure;
 *   - no CUDA or torch types: device pointers are plain pointers obtained from
 *     nmx_malloc (or any cudaMalloc'd memory of the context's device);
 *   - addresses are uint32 (the reference's 9-byte packet record already limits
 *     them to 32 bits, traffic.py:25,370-372); `address_space` is 1..2^32;
 *   - a `valid` column is optional (NULL = all valid), one byte per packet,
 *     nonzero = valid (traffic.py:43-51);
 *   - statistics are int64 in this order (the "stats9" layout):
 *       0 valid_packets        1 unique_links        2 max_link_packets
 *       3 unique_sources       4 max_source_packets  5 max_fanout
 *       6 unique_destinations  7 max_destination_packets  8 max_fanin
 *     (analytics.py:31-40 AggregateReport + the three Graph Challenge maxima);
 *   - one context = one device + one CUDA stream; calls on one context are
 *     serialised by an internal lock, so a context may be shared by threads
 *     (tests/test_analytics.py:178-194).
 */
#ifndef NMX_H
#define NMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMX_OK 0
#define NMX_EINVAL -1  /* maps to ValueError / TypeError in Python */
#define NMX_ENOMEM -2  /* device or pinned-host allocation failed  */
#define NMX_ECUDA -3   /* CUDA runtime / kernel error              */
#define NMX_ENODEV -4  /* no CUDA device                           */

#define NMX_GEN_UNIFORM 0  /* SURVEY.md 8(d) cfg3 generator */
#define NMX_GEN_POWERLAW 1 /* SURVEY.md 8(d) cfg4 "octave" generator */

#define NMX_REDUCE_SUM 0 /* analytics.py:84-86 sum_reduce (int64 wrap) */
#define NMX_REDUCE_MAX 1 /* analytics.py:89-92 max_scan (INT64_MIN sentinel -> 0) */

typedef struct nmx_ctx nmx_ctx;
typedef struct nmx_coo nmx_coo;

int nmx_version(void);
const char* nmx_last_error(void);
int nmx_device_count(int* count);

/* Execution resource: replaces one member pool of make_group_scheduler
 * (resources.py:139-159); resource_count == number of contexts. */
int nmx_create(int device, nmx_ctx** out);
void nmx_destroy(nmx_ctx* ctx);
/* the context's cudaStream_t, as an opaque pointer (for interop only) */
void* nmx_stream(nmx_ctx* ctx);
int nmx_synchronize(nmx_ctx* ctx);

/* device / pinned memory owned by the caller */
int nmx_malloc(nmx_ctx* ctx, uint64_t bytes, void** dptr);
int nmx_free(nmx_ctx* ctx, void* dptr);
int nmx_host_alloc(uint64_t bytes, void** hptr);
int nmx_host_free(void* hptr);
int nmx_memcpy_h2d(nmx_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int nmx_memcpy_d2h(nmx_ctx* ctx, void* dst, const void* src, uint64_t bytes);

/* Synthetic packets i in [offset, offset+n) of stream `seed` into device
 * columns; chunk-addressable. Same integer function as oracle/netmeter_oracle.py
 * gen_uniform / gen_powerlaw. (Input preparation, cf. traffic.py:82-104.) */
int nmx_generate(nmx_ctx* ctx, int kind, uint64_t seed, uint64_t offset, uint64_t n, uint64_t address_space,
                 uint32_t* d_src, uint32_t* d_dst);

/* THE HOT PATH. Nine statistics of the traffic matrix summed over all valid
 * packets, i.e. build_matrices(stream, window_size=len(stream)) (traffic.py:221-242)
 * -> to_flat (traffic.py:263-292) -> analyze_matrix (analytics.py:95-106)
 * + max_scan over weights / row_sums[:,1] / col_sums[:,1] (analytics.py:89-92).
 * Device-resident columns; n < 2^32 per call. */
int nmx_stats9_device(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                      uint64_t address_space, int64_t out[9]);
/* Same, from host columns (copied H2D inside the call; pinned memory is fastest). */
int nmx_stats9_host(nmx_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                    uint64_t address_space, int64_t out[9]);
/* A sequence of independent host batches (src[k], dst[k], valid[k] or NULL, lens[k]
 * packets each < 2^32; pinned memory streams at full host-link bandwidth): batch k's
 * nine statistics -> out[9k .. 9k+8], each exactly nmx_stats9_host of that batch.
 * Batch k+1's H2D copy (second stream, two device slots) overlaps batch k's device
 * work, so a run of batches is bound by the host link rather than by copy + compute.
 * The loop the reference writes as repeated analyze_matrix calls over packet windows
 * (analytics.py:95-130); host buffers are borrowed until the call returns. */
int nmx_stats9_host_batches(nmx_ctx* ctx, uint64_t nbatch, const uint32_t* const* src, const uint32_t* const* dst,
                            const uint8_t* const* valid, const uint64_t* lens, uint64_t address_space, int64_t* out);
/* Same, from the reference's own PacketStream columns (traffic.py:43-71: int64 src /
 * dst, bool valid as bytes, any host memory): narrowed to u32 by host threads into
 * pinned slots window by window, overlapped with the copies and the device work.
 * Addresses outside [0, address_space) -> NMX_EINVAL. */
int nmx_stats9_host_i64(nmx_ctx* ctx, const int64_t* src, const int64_t* dst, const uint8_t* valid, uint64_t n,
                        uint64_t address_space, int64_t out[9]);

/* Streamed windows (BASELINE config 5): nine statistics of the matrix summed over
 * `nwin` windows of HOST packet columns (src[k], dst[k], valid[k] or NULL, lens[k]
 * packets; pinned memory for full host-link bandwidth), i.e. the cross-window sum
 * A = sum_t A_t = build_matrices(concatenation, window_size=total) (traffic.py:221-242).
 * The H2D copy of window k+1 overlaps the device work of window k (two streams);
 * the total must be < 2^32 packets per device. valid may be NULL (all valid). */
int nmx_stream_stats9(nmx_ctx* ctx, const uint32_t* const* src, const uint32_t* const* dst,
                      const uint8_t* const* valid, const uint64_t* lens, uint64_t nwin, uint64_t address_space,
                      int64_t out[9]);

/* Packet files: the reference's binary records, 9 bytes each,
 * little-endian {u32 src, u32 dst, u8 valid} (traffic.py:25 _PACKET_DTYPE,
 * write_packets / read_packets traffic.py:370-388).
 *  - nmx_stream_records: like nmx_stream_stats9 over windows of HOST records
 *    (rec[k], lens[k] records), streamed raw (9 B/packet) and unpacked on the device.
 *  - nmx_unpack_records: device records -> device columns (d_rec 4-byte aligned,
 *    d_src / d_dst 16-byte, d_valid 4-byte aligned).
 * Both reject any address >= address_space with NMX_EINVAL, as PacketStream does
 * (traffic.py:56-64). */
int nmx_stream_records(nmx_ctx* ctx, const uint8_t* const* rec, const uint64_t* lens, uint64_t nwin,
                       uint64_t address_space, int64_t out[9]);
int nmx_unpack_records(nmx_ctx* ctx, const uint8_t* d_rec, uint64_t n, uint32_t* d_src, uint32_t* d_dst,
                       uint8_t* d_valid, uint64_t address_space);

/* anonymize (traffic.py:107-137) on the device: every address of
 * the interleaved stream src0, dst0, src1, dst1, ... is relabelled with
 * perm[first-seen rank], perm = numpy default_rng(key).permutation(k) drawn by the
 * caller once k (the number of distinct addresses) is known. Two calls:
 *  - nmx_anonymize_begin: device columns (n < 2^31 packets) -> k; the sorted
 *    state stays in the context (one anonymization per context at a time);
 *  - nmx_anonymize_finish: host perm[k] (u32) -> relabelled device columns, and
 *    optionally the host tables distinct_out[k] (ascending raw addresses) and
 *    code_out[k] (their codes) of the AnonymizationMap. */
int nmx_anonymize_begin(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t* k_out);
int nmx_anonymize_finish(nmx_ctx* ctx, const uint32_t* perm, uint32_t* d_src_out, uint32_t* d_dst_out,
                         uint32_t* distinct_out, uint32_t* code_out);

/* Text matrix files (traffic.py:295-367): header "dim nnz", then
 * "row col value" lines sorted row-major without duplicates.
 *  - nmx_parse_matrix_text: host text -> device COO (keys row << 32 | col, int64 values),
 *    tokenised, converted and validated on the device with the reference's rules
 *    (str.splitlines / str.split / int(), int64 entries) and its check order. info[8]:
 *    [0] dim, [1] nnz (header), [2] entry lines, [3] NMX_TXT_* diagnosis (0 = parsed,
 *    *out set), [4] the 1-based physical line it names (0 = none). A malformed file is
 *    NMX_OK with info[3] != 0 (the caller words the MatrixFileError); NMX_TXT_ENCODING
 *    asks the caller to normalise non-ASCII text (str.split semantics) and call again;
 *    NMX_TXT_WIDE = dim > 2^32 (rows / columns beyond the 32-bit key halves).
 *  - nmx_format_matrix_text: entry columns -> the "row col value\n" lines (without the
 *    header); call with out == NULL (or cap too small) to get *bytes first. */
#define NMX_TXT_OK 0
#define NMX_TXT_HEADER 1    /* "expected header 'dim nnz'" */
#define NMX_TXT_DIM 2       /* "dim must be >= 1" */
#define NMX_TXT_NNZ 3       /* "nnz must be >= 0" */
#define NMX_TXT_FIELDS 4    /* "expected 'row col value'" */
#define NMX_TXT_INTEGERS 5  /* "expected 'row col value' integers" */
#define NMX_TXT_COUNT 6     /* "header claims {nnz} entries, file has {k}" */
#define NMX_TXT_BOUNDS 7    /* "row/col outside [0, {dim})" */
#define NMX_TXT_VALUE 8     /* "value must be >= 1" */
#define NMX_TXT_ORDER 9     /* "entries must be sorted row-major with no duplicates" */
#define NMX_TXT_WIDE 10
#define NMX_TXT_ENCODING 11
int nmx_parse_matrix_text(nmx_ctx* ctx, const char* text, uint64_t bytes, int64_t info[8], nmx_coo** out);
int nmx_format_matrix_text(nmx_ctx* ctx, const int64_t* rows, const int64_t* cols, const int64_t* vals, uint64_t nnz,
                           char* out, uint64_t cap, uint64_t* bytes);

/* Per-window statistics: window t = packets [t*W, (t+1)*W) by raw position,
 * invalid packets keep their position (traffic.py:221-242); out has
 * ceil(n/W) rows of 9 (analyze_dataset per-window reports, analytics.py:109-130). */
int nmx_window_stats9_device(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                             uint64_t n, uint64_t address_space, uint64_t window_size, int64_t* out);
int nmx_window_stats9_host(nmx_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                           uint64_t address_space, uint64_t window_size, int64_t* out);

/* Reductions of the drop-in sum_reduce / max_scan (analytics.py:54-92) over a
 * host int64 view: op NMX_REDUCE_SUM wraps mod 2^64; NMX_REDUCE_MAX returns
 * INT64_MIN for an empty view (the Python layer maps it to 0). */
int nmx_reduce_i64(nmx_ctx* ctx, const int64_t* data, uint64_t n, int op, int64_t* out);

/* Materialisation for the drop-in containers:
 *  - nmx_coo_build: sorted unique links of host packets with counts, i.e.
 *    np.unique(src*dim+dst, return_counts=True) (traffic.py:207), per window
 *    when window_size > 0 (build_matrices, traffic.py:221-242). Keys are
 *    packed as window<<2b | src<<b | dst with b = ceil(log2(address_space));
 *    requires 2b + window bits <= 64. Kept in the context until the next call;
 *  - nmx_coo_fetch: copy keys / counts of the last nmx_coo_build to the host;
 *  - nmx_coo_rowptr: dense row_ptr[dim+1] of the COO slice [lo, hi) of one
 *    window (traffic.py:210-211);
 *  - nmx_flat_build / nmx_flat_fetch: to_flat (traffic.py:263-292) of a CSR
 *    matrix: per-nonzero row ids (edges[:,0]), occupied rows with nnz (fan-out)
 *    and value sums, occupied columns with nnz (fan-in) and value sums. Values
 *    must lie in [1, 2^32) (packet counts); nnz, dim < 2^32. */
int nmx_coo_build(nmx_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                  uint64_t address_space, uint64_t window_size, uint64_t* nnz);
int nmx_coo_fetch(nmx_ctx* ctx, uint64_t* keys, int64_t* counts);
int nmx_coo_rowptr(nmx_ctx* ctx, uint64_t lo, uint64_t hi, uint64_t window, uint64_t dim, int64_t* row_ptr);
int nmx_flat_build(nmx_ctx* ctx, const int64_t* row_ptr, uint64_t dim, const int64_t* col_idx, const int64_t* values,
                   uint64_t nnz, uint64_t* rows_out, uint64_t* cols_out);
int nmx_flat_fetch(nmx_ctx* ctx, int64_t* edge_src, int64_t* row_ids, int64_t* row_nnz, int64_t* row_sum,
                   int64_t* col_ids, int64_t* col_nnz, int64_t* col_sum);

/* Sorted unique COO matrices on the device and their element-wise sum (SURVEY.md
 * 8(a) a11, the merge-path "K10"): keys are (src<<32)|dst, counts u64 in [1, 2^63)
 * (the reference's int64 matrix values). The
 * summed matrix of several windows is merge_add of their COOs (= the matrix of
 * the concatenated packets, traffic.py:221-242 with one window).
 *  - nmx_coo_from_packets: unique links of device packet columns;
 *  - nmx_coo_merge_add: C = A + B by merge path (counts of shared keys added; a sum
 *    beyond 2^63 - 1 is NMX_EINVAL);
 *  - nmx_coo_stats9: the nine statistics of a COO (counts >= 2^32 take 64-bit hash
 *    tables, up to 2^28 links);
 *  - nmx_coo_nnz / nmx_coo_download / nmx_coo_free;
 *  - nmx_coo_reserve: keep `bytes` of device memory mapped in the pool COOs are
 *    allocated from (stream-ordered allocations then never grow the pool). */
int nmx_coo_from_packets(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                         uint64_t n, nmx_coo** out);
int nmx_coo_merge_add(nmx_ctx* ctx, const nmx_coo* a, const nmx_coo* b, nmx_coo** out);
/* host sorted unique keys (src << 32 | dst) + counts >= 1 -> device COO */
int nmx_coo_upload(nmx_ctx* ctx, const uint64_t* keys, const int64_t* counts, uint64_t nnz, nmx_coo** out);
int nmx_coo_stats9(nmx_ctx* ctx, const nmx_coo* a, int64_t out[9]);
int nmx_coo_nnz(const nmx_coo* a, uint64_t* nnz);
int nmx_coo_download(nmx_ctx* ctx, const nmx_coo* a, uint64_t* keys, int64_t* counts);
void nmx_coo_free(nmx_coo* a);
int nmx_coo_reserve(nmx_ctx* ctx, uint64_t bytes);

/* Multi-GPU building blocks (one process per GPU; the exchange itself is NCCL
 * all-to-all driven by paper_2510_14050_b200/distributed.py). owner(x) =
 * (fmix32(x) * nparts) >> 32, nparts <= 64. Counts are written to host arrays.
 *  - nmx_partition_packets: route valid packets by owner(src) into
 *    part-contiguous output columns (capacity n each);
 *  - nmx_shard_rows: link + row statistics of packets whose sources this rank
 *    owns (fields 0-5 of stats9 exact; 6-8 zero) and its unique links' (dst,
 *    count) column entries routed by owner(dst) (capacity n each);
 *  - nmx_shard_cols: column statistics (fields 6-8) of received column entries.
 * No reference counterpart: the reference is single-process. */
int nmx_partition_packets(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                          uint64_t n, int nparts, uint32_t* d_out_src, uint32_t* d_out_dst, uint64_t* counts);
int nmx_shard_rows(nmx_ctx* ctx, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t address_space,
                   int nparts, uint32_t* d_out_dst, uint32_t* d_out_count, uint64_t* counts, int64_t out[9]);
int nmx_shard_cols(nmx_ctx* ctx, const uint32_t* d_dst, const uint32_t* d_count, uint64_t u, uint64_t address_space,
                   int64_t out[9]);

/* Device groups: one process driving G ranks, each an nmx_ctx (own stream and
 * workspace) on devices[r] -- the B200 counterpart of make_group_scheduler(G)
 * (resources.py:139-159), whose resource_count is G. Several ranks may name the same
 * device (virtual ranks). The summed-matrix statistics of a group run the sharded
 * pipeline of SURVEY.md 8(e) inside the library, one host thread per rank:
 * valid packets to owner(src) = (fmix32(src) * G) >> 32, links + rows locally, unique
 * links' (dst, count) to owner(dst), columns locally, SUM / MAX combine. Both
 * all-to-all exchanges are peer copies (cudaMemcpyPeerAsync over NVLink / NVSwitch
 * between distinct devices, with peer access enabled at creation) ordered by
 * cross-stream events; bit-identical to one device for every G.
 *  - nmx_group_stats9_device: rank r's n[r] packets are device columns of devices[r];
 *  - nmx_group_stats9_host: one host stream split by partition_even into G spans
 *    (partitioning.py:62-70), each copied to its rank in batch_count chunks (the
 *    reference's b_n sub-batches, partitioning.py:89-98);
 *  - nmx_group_context: rank r's context (for nmx_malloc etc. on its device);
 *  - nmx_group_last_exchange: bytes moved by the last call's two exchanges. */
typedef struct nmx_group nmx_group;
int nmx_group_create(const int* devices, int g, nmx_group** out);
void nmx_group_destroy(nmx_group* grp);
int nmx_group_size(const nmx_group* grp, int* g);
int nmx_group_context(nmx_group* grp, int rank, nmx_ctx** out);
int nmx_group_stats9_device(nmx_group* grp, const uint32_t* const* d_src, const uint32_t* const* d_dst,
                            const uint8_t* const* d_valid, const uint64_t* n, uint64_t address_space, int64_t out[9]);
int nmx_group_stats9_host(nmx_group* grp, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                          uint64_t address_space, uint64_t batch_count, int64_t out[9]);
int nmx_group_last_exchange(nmx_group* grp, uint64_t* bytes1, uint64_t* bytes2);

/* NCCL communicators: the multi-process form (one process per GPU, the driver's
 * torchrun launch) of the same sharded pipeline. Rank 0 makes an id with
 * nmx_comm_unique_id and hands it to every rank out of band (bytes); each rank calls
 * nmx_comm_init on its context (collective). nmx_stats9_sharded[_host] runs exchange 1
 * (valid packets to owner(src)), links + rows, exchange 2 ((dst, count) of unique links
 * to owner(dst)), columns and the SUM / MAX combine inside the library: grouped
 * ncclSend / ncclRecv on the context stream for both all-to-alls, ncclAllGather for
 * the part counts, two ncclAllReduce for the statistics. Every rank gets the nine
 * statistics of the matrix summed over all ranks' packets (bit-identical to one
 * device). Replaces the reference's make_group_scheduler(G) fan-out
 * (resources.py:139-159, analytics.py:68-81) across processes. */
#define NMX_COMM_ID_BYTES 128
typedef struct nmx_comm nmx_comm;
int nmx_comm_unique_id(uint8_t* id);
int nmx_comm_init(nmx_ctx* ctx, const uint8_t* id, int nranks, int rank, nmx_comm** out);
void nmx_comm_destroy(nmx_comm* comm);
int nmx_stats9_sharded(nmx_ctx* ctx, nmx_comm* comm, const uint32_t* d_src, const uint32_t* d_dst,
                       const uint8_t* d_valid, uint64_t n, uint64_t address_space, int64_t out[9]);
int nmx_stats9_sharded_host(nmx_ctx* ctx, nmx_comm* comm, const uint32_t* src, const uint32_t* dst,
                            const uint8_t* valid, uint64_t n, uint64_t address_space, int64_t out[9]);
int nmx_comm_last_exchange(nmx_comm* comm, uint64_t* bytes1, uint64_t* bytes2);

/* Timing hooks used by bench.py: CUDA-event time (ms) of the last hot-path
 * call's whole device section, and of its sort / partition section (the MSD
 * row partition, or the onesweep passes on the LSD path) summed over launches,
 * plus the number of kernels it launched. */
int nmx_last_timing(nmx_ctx* ctx, float* total_ms, float* sort_ms, int* sort_launches, int* kernel_launches);
/* Per-stage CUDA-event times (ms) of the last hot-path call. MSD path (7): [0] setup,
 * [1] row partition, [2] row groups, [3] heavy rows, [4] column partition,
 * [5] column groups, [6] heavy columns + result copy. LSD path (5): [0] ingest
 * histogram (+ host pass planning), [1] row sort (onesweep passes), [2] fused
 * link/row kernel, [3] column sort, [4] column kernel + result copy. Returns the count. */
int nmx_last_stages(nmx_ctx* ctx, float* ms, int cap);
/* The dominant kernel class of the last hot-path call (the MSD partition scatter,
 * or the onesweep pass on the LSD path): summed CUDA-event time of its launches,
 * launch count, algorithmic bytes (item bytes in + out per launch: 16 per item on
 * the u64 levels, 12 on the column level that narrows items to u32, 8 on the u32
 * levels) and name. */
int nmx_last_kernel_class(nmx_ctx* ctx, float* ms, int* launches, uint64_t* bytes, char* name, int name_cap);
/* The same class launch by launch (up to cap): CUDA-event ms and algorithmic bytes
 * of each; *count = the number of launches recorded (<= 32). */
int nmx_last_kernel_launches(nmx_ctx* ctx, int cap, float* ms, uint64_t* bytes, int* count);

#ifdef __cplusplus
}
#endif

#endif /* NMX_H */
