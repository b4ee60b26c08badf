/*
 * nest.h -- C ABI of libnest.so, the B200 (sm_100a) hot path of NestPipe
 * (arXiv 2604.06956): the synchronous row-sharded embedding step, forward and
 * backward, with Dual-Buffer Pipelining (DBP) and Frozen-Window Pipelining
 * (FWP).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (the reference's
 * documents), SURVEY = /root/repo/SURVEY.md section.  Every entry point states
 * the passage that defines the operation it performs.
 *
 * Conventions (apply to every call unless stated otherwise)
 * -----------------------------------------------------------------------
 * Keys      int64 packed (table << 40) | row, row < table_rows[table]
 *           (SURVEY Q2).  Owner of a key = row mod world, local row inside
 *           the owner's shard of that table = row div world (Q1).
 * Batches   CSR, sample-major: bag (b, f) = b*F + f holds the keys sample b
 *           has for feature f; bag_offsets is int32[B*F+1].
 * Shard     the rank's slice of every table, rows (table, local row)
 *           concatenated table by table, fp32 [shard_rows, dim], in the
 *           caller-owned `table_mem` (tables row-sharded, the HBM
 *           shard plays the role of the host store written back to).
 * Memory    every device byte is owned by the caller: query sizes with
 *           nest_workspace_bytes, pass device pointers (e.g. torch tensors).
 *           The library owns only its NCCL communicators (when given ids),
 *           the exchange windows (W > 1: peer-mapped row / count / key areas
 *           and flags), CUDA events, two internal streams (the occurrence
 *           sorts, the tower's dW GEMMs; replaceable, nest_set_streams) and
 *           small pinned host mirrors.  Pointers are device pointers unless
 *           marked "host".  Inputs are read-only.
 * Streams   `void*` arguments named *stream / compute / comm are cudaStream_t
 *           (NULL = the legacy default stream).  All calls are
 *           stream-asynchronous except nest_route / nest_route_end (one host
 *           sync for the All2All sizes), nest_create,
 *           nest_destroy, nest_set_streams and the read-back helpers.
 * Slots     two pipeline slots (0/1) hold the per-batch state: routing
 *           results and one HBM buffer each; their roles (active/prefetch)
 *           alternate every step.
 * Errors    host-detectable errors return immediately and leave the context
 *           unchanged.  Device-detected errors (key out of range, foreign key
 *           at an owner) are raised at the next nest_route(_end) sync, become
 *           sticky, and every later call returns that code (CUDA-style).
 *           Calls never abort or throw.  nest_last_error gives a message.
 *           Collective consistency: the count exchange carries every rank's
 *           error flags and counts to every rank, so all ranks take the same
 *           error decision at the same call.
 */
#ifndef NEST_H_
#define NEST_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NEST_API __attribute__((visibility("default")))
#else
#define NEST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NEST_OK = 0,
  NEST_ERR_INVALID = 1,       /* bad argument / shape / config (SPEC exit 2) */
  NEST_ERR_CUDA = 2,          /* a CUDA runtime call failed */
  NEST_ERR_NCCL = 3,          /* an NCCL call failed */
  NEST_ERR_CAPACITY = 4,      /* counts exceed a preallocated capacity */
  NEST_ERR_KEY_RANGE = 5,     /* table >= num_tables or row >= table_rows */
  NEST_ERR_SHARD = 6,         /* owner received a key it does not own */
  NEST_ERR_ORDER = 7,         /* call out of order: e.g. lookup before route */
  NEST_ERR_DIVISIBILITY = 8   /* B mod N != 0 */
} nest_status_t;

typedef struct nest_ctx nest_ctx_t;   /* opaque; one per rank */

enum { NEST_POOL_SUM = 0, NEST_POOL_NONE = 1 };
enum { NEST_INIT_UNIFORM = 0, NEST_INIT_DYADIC = 1, NEST_INIT_ZERO = 2 };
enum { NEST_SCHED_SEQUENTIAL = 0, NEST_SCHED_CLUSTERED = 1 };
/* sparse optimizer of the update: SGD of Eq. 2, or row-wise
 * AdaGrad (the paper and SPEC leave it open) */
enum { NEST_OPT_SGD = 0, NEST_OPT_ROWWISE_ADAGRAD = 1 };
/* where the table shard lives (nest_config_t.table_location) */
enum { NEST_TABLE_HBM = 0, NEST_TABLE_HOST = 1 };
enum { NEST_MAX_WORLD = 64, NEST_MAX_MICRO_BATCHES = 8, NEST_MAX_TABLES = 1024 };

/* Static configuration of one rank.  Capacities bound every per-batch count;
 * 0 selects the documented default. */
typedef struct {
  int32_t world;              /* W >= 1 ranks (one per GPU) */
  int32_t rank;               /* 0 <= rank < W */
  int32_t num_tables;         /* T <= NEST_MAX_TABLES */
  int32_t dim;                /* d in {16, 32, 64, 128, 256} (fp32 rows) */
  const int64_t* table_rows;  /* host [T]: rows of every table */
  int32_t pooling;            /* NEST_POOL_SUM or NEST_POOL_NONE (expand) */
  int32_t num_features;       /* F >= 1 bags per sample */
  int64_t max_keys;           /* K cap: key occurrences per rank per batch (< 2^28) */
  int64_t max_batch;          /* B cap: samples per rank per batch */
  int32_t max_micro_batches;  /* N cap, 1..NEST_MAX_MICRO_BATCHES */
  int64_t max_recv_keys;      /* R_o cap: keys an owner receives per batch (default max_keys at W=1,
                                 min(2, W) * max_keys otherwise); sizes the owner buffers */
  int64_t max_owner_keys;     /* reserved (U_o cap is derived: min(max_recv_keys, shard rows)) */
  int64_t max_mb_rows;        /* cap of sum_i U_{s,i} (rows a source receives over all micro-batches; default max_keys) */
  int64_t max_owner_mb_rows;  /* cap of sum_i R_{o,i} (rows an owner sends over all micro-batches; default max_recv_keys*N clamped) */
  uint64_t seed;              /* PRF seed of the table initialisation */
  int32_t init_mode;          /* NEST_INIT_UNIFORM (+-1/sqrt(d)), _DYADIC (parity regime P1), _ZERO */
  int32_t tower_layers;       /* stand-in dense tower depth L (0 = no tower) */
  int32_t tower_hidden;       /* tower width (bf16 GEMMs) */
  int32_t optimizer;          /* NEST_OPT_SGD (default) or NEST_OPT_ROWWISE_ADAGRAD */
  float adagrad_eps;          /* AdaGrad denominator epsilon (fp32) */
  int32_t table_location;     /* NEST_TABLE_HBM (default): table_mem is device memory.
                                 NEST_TABLE_HOST: table_mem is pinned host memory (cudaHostAlloc /
                                 cudaHostRegister, device-accessible through UVA) -- the host-DRAM
                                 tier of SURVEY §8(f) NEXT-3: the DBP
                                 retrieval (R4 prefetch gather, R5 refresh) reads rows over PCIe
                                 into the HBM slot buffers, the write-back (R12) stores them back;
                                 everything else stays in HBM.  nest_create checks the pointer
                                 kind and returns NEST_ERR_INVALID on a mismatch. */
  int32_t tower_train;        /* 0 (default): the stand-in tower is fixed (north_star).  1: trained
                                 (P:461-462 dense gradients AllReduced on the
                                 communication side): the weight-gradient GEMMs of every tower call
                                 of a batch (one per micro-batch) accumulate into one fp32 dW, so
                                 all micro-batches of the window see the same frozen weights
                                 (Prop. 2, Corollary 1); nest_tower_step then sums dW
                                 over the ranks (ncclAllReduce on a communicator split from the
                                 window's) and applies W -= tower_lr * sum_r dW_r to fp32 master
                                 weights (bf16 copies feed the GEMMs) once, on the library's dW
                                 stream; the next tower call waits for it.  Collective: every rank
                                 makes the same sequence of nest_tower_fwd_bwd* / nest_tower_step
                                 calls. */
  float tower_lr;             /* step size of the trained tower (fp32) */
} nest_config_t;

/* Host-known counts of one slot after nest_route (all per this rank). */
typedef struct {
  int32_t valid;              /* 1 after a successful nest_route on the slot */
  int32_t num_micro_batches;  /* N of the routed batch */
  int32_t batch;              /* B */
  int64_t nnz;                /* K key occurrences */
  int64_t uniq;               /* U_s source-unique keys (sum of send counts) */
  int64_t recv;               /* R_o keys received as owner */
  int64_t mb_uniq[NEST_MAX_MICRO_BATCHES];   /* U_{s,i}: rows received in mb i */
  int64_t mb_recv[NEST_MAX_MICRO_BATCHES];   /* R_{o,i}: rows sent as owner in mb i */
  int64_t mb_nnz[NEST_MAX_MICRO_BATCHES];    /* K_i occurrences in mb i */
  int64_t mb_out_rows[NEST_MAX_MICRO_BATCHES]; /* rows of `out`/`dout` for mb i */
} nest_slot_info_t;

/* Device pointers into a slot's routing results (for parity checks). */
typedef struct {
  const int64_t* uniq;        /* [U_s] unique keys, (owner, key) ascending */
  const int32_t* inverse;     /* [K] uniq[inverse[j]] == keys[j] */
  const uint32_t* mask;       /* [U_s] bit i set iff the key occurs in micro-batch i */
  const int32_t* pos;         /* [N][U_s+1] index of u among mask-bit-i keys */
  const int32_t* send_counts; /* [W][Nm+2], Nm = max_micro_batches: per owner
                                 {U, U_1..U_N, (unused up to Nm), err} */
  const int32_t* all_counts;  /* [W][W][Nm+2] every rank's send_counts (count exchange) */
  const int64_t* recv_keys;   /* [R_o] received keys | mask << 56, sources concatenated */
  const int32_t* owner_rows;  /* [U_o] shard row of every owner-unique key, ascending */
  const int32_t* owner_inv;   /* [R_o] owner-unique index of every received key */
  const int32_t* n_owner;     /* [1] U_o */
  const float* buffer;        /* [U_o][d] the slot's HBM buffer (active or prefetch) */
} nest_route_view_t;

/* Library version string. */
NEST_API const char* nest_version(void);

/* Writes a 128-byte NCCL unique id into uid_out (host memory).  Call on rank 0
 * twice (main + aux communicator) and broadcast the bytes to all ranks. */
NEST_API nest_status_t nest_get_unique_id(void* uid_out);

/* Bytes of table memory (the shard, fp32 [shard_rows, dim], then with
 * NEST_OPT_ROWWISE_ADAGRAD the fp32 accumulators [shard_rows]) and of
 * workspace this configuration needs.  Pure host computation. */
NEST_API nest_status_t nest_workspace_bytes(const nest_config_t* cfg, size_t* table_bytes,
                                   size_t* work_bytes);

/* Number of shard rows this rank stores: sum_t |{row < rows_t : row mod W = rank}|. */
NEST_API int64_t nest_shard_rows(const nest_config_t* cfg);

/* Creates a context.  nccl_uids: host, 2 x 128 bytes (main and aux
 * communicator) from nest_get_unique_id on rank 0 -- collective over all ranks
 * (ncclCommInitRank), the exchange windows are connected through NCCL -- or
 * NULL.  NULL with world == 1: no communication at all.  NULL with world > 1:
 * no NCCL (every exchange of the path -- count exchange, key All2All (R2),
 * embedding and gradient All2All (R7, R11), the trained tower's dense
 * AllReduce -- runs over the peer-mapped exchange windows, P:343, P:349,
 * P:354); the caller then connects the ranks with nest_window_export /
 * nest_window_connect before the first nest_route.  That mode also runs
 * several ranks on ONE device (in one process or several): the peers' windows
 * are plain device memory there.  It needs the fused or ce transport
 * (NEST_A2A != nccl), else NEST_ERR_INVALID.  table_mem / work_mem: device
 * buffers of at least the queried sizes, 256-byte aligned.  On failure every
 * resource already created is released. */
NEST_API nest_status_t nest_create(const nest_config_t* cfg, const void* nccl_uids,
                          void* table_mem, void* work_mem, void* stream,
                          nest_ctx_t** out);
NEST_API nest_status_t nest_destroy(nest_ctx_t* ctx);

/* Checked mode (environment NEST_GUARD=1 when the context is sized and
 * created): every workspace buffer is followed by a 256-byte guard band filled
 * with a pattern at nest_create; this call counts the guard words that no
 * longer hold it, i.e. out-of-bounds writes into the workspace since creation
 * (a substitute for compute-sanitizer memcheck, unavailable on the GPU pool).
 * Enqueued on `stream` after its work, then synchronises it.  *bad_words = 0
 * when every band is intact.  NEST_ERR_INVALID outside checked mode. */
NEST_API nest_status_t nest_check_guards(nest_ctx_t* ctx, void* stream, int64_t* bad_words);

/* Exchange-window record of one rank (host bytes; plain data the caller moves
 * between ranks with any transport, e.g. torch.distributed.all_gather_object):
 * the window's device pointer and CUDA IPC handle plus its geometry. */
typedef struct {
  uint64_t magic;
  int32_t pid, rank, world, device;
  uint64_t ptr;                  /* device address (used directly by same-process peers) */
  uint8_t ipc[64];               /* cudaIpcMemHandle_t (other processes) */
  uint64_t bytes, off_own, off_cnt, off_key, off_twr, off_flags;
  uint64_t src_stride, cnt_stride, key_stride;
  /* direct write-back (W > 1, fused transport, SGD, HBM tables): the owner
   * marks every row it pushes with the row's shard index when the requester is
   * the key's only contributor (one source, one micro-batch), and that
   * requester applies Eq. 2 to its received copy and stores the updated row
   * straight into the owner's shard -- so the shard is mapped too */
  uint64_t off_dwb, dwb_stride;  /* int32 marks, per slot, indexed like the receive rows */
  uint64_t shard_ptr, shard_off; /* shard device address; its offset in the IPC-mapped allocation */
  uint8_t shard_ipc[64];         /* cudaIpcMemHandle_t of the allocation holding the shard */
  int32_t dwb_ok, dwb_pad;       /* 1: this rank can take part (the feature runs iff every rank can) */
} nest_window_rec_t;

/* This rank's window record (context created with nccl_uids == NULL and
 * world > 1).  rec: host, sizeof(nest_window_rec_t).  NEST_ERR_INVALID when the
 * context has no window. */
NEST_API nest_status_t nest_window_export(const nest_ctx_t* ctx, nest_window_rec_t* rec);

/* Maps every rank's window (recs: host, world records in rank order, from
 * nest_window_export on each rank).  Same-process peers are addressed
 * directly, others through cudaIpcOpenMemHandle.  Host-side only; call once,
 * on every rank, before the first nest_route.  NEST_ERR_INVALID on records of
 * another world / geometry, NEST_ERR_ORDER if already connected. */
NEST_API nest_status_t nest_window_connect(nest_ctx_t* ctx, const nest_window_rec_t* recs);

/* PRF initialisation of the whole shard: row of key k gets init_row(seed, k,
 * d). */
NEST_API nest_status_t nest_init_tables(nest_ctx_t* ctx, void* stream);

/* FWP partition of the local batch into N equal micro-batches (
 * S:544-552; SURVEY §8(c) clustering spec).  mode NEST_SCHED_SEQUENTIAL slices
 * by sample id; NEST_SCHED_CLUSTERED runs the round-based key-centric greedy.
 * Outputs: perm_out int32[B] (samples of micro-batch i are
 * perm_out[mb_offsets_out[i] .. mb_offsets_out[i+1]), ascending id inside a
 * micro-batch), mb_offsets_out int32[N+1].  B mod N != 0 -> NEST_ERR_DIVISIBILITY.
 * keys / bag_offsets / nnz: the local batch (unused by SEQUENTIAL).  Issue it
 * on the same stream as the following nest_route (they share scratch).
 * CLUSTERED needs B < 2^21 and at most 16,383 distinct keys per sample. */
NEST_API nest_status_t nest_fwp_schedule(nest_ctx_t* ctx, const int64_t* keys,
                                const int32_t* bag_offsets, int64_t nnz, int32_t B, int32_t N,
                                int32_t mode, int32_t* perm_out,
                                int32_t* mb_offsets_out, void* stream);

/* Key Routing + Embedding Retrieval of DBP for one
 * batch into `slot`: source dedup and owner bucketing, exchange of counts (one
 * host sync), key All2All, owner dedup, gather of the owned rows from the
 * shard into the slot's HBM buffer.  keys/bag_offsets: the local batch (nnz
 * occurrences, B samples).  perm/mb_offsets from nest_fwp_schedule (NULL =
 * one micro-batch, N must be 1).  The gather is ordered after this slot's
 * previous update's write-back (events inside the library, reading Q8).  If
 * the other slot is routed and its update is still to come (the pipelined
 * call order: route(t+1) inside window t), the gather skips that slot's keys
 * K(t) -- they are supplied, updated, by nest_dbp_refresh, which then becomes
 * mandatory before any lookup of this slot (NEST_ERR_ORDER otherwise) -- so
 * the retrieval never waits for the update of window t.  Otherwise the gather
 * waits for the other slot's update.  With the
 * fused NVLink transport (world > 1, NEST_A2A unset, NEST_EARLY_PUSH != 0)
 * the owner then pushes every requested row of the buffer into the
 * requesters' receive rows of this slot (the embedding All2All, issued here
 * on `stream` instead of inside the window). */
NEST_API nest_status_t nest_route(nest_ctx_t* ctx, int32_t slot, const int64_t* keys,
                         const int32_t* bag_offsets, int64_t nnz, int32_t B,
                         const int32_t* perm, const int32_t* mb_offsets, int32_t N,
                         void* stream);

/* nest_route in two halves, so the caller's thread is not blocked while it
 * still has window work to enqueue.  nest_route_begin enqueues the source
 * side (dedup, owner bucketing, masks, the count exchange and its copy to the
 * host) on `stream` and returns; nest_route_end performs the one host sync
 * (the counts), then enqueues the rest (key All2All, owner dedup, gather,
 * early push, occurrence sort) on the same stream.  Between the two no other
 * nest_route_begin / nest_fwp_schedule may be issued (they share the routing
 * scratch: NEST_ERR_ORDER) and the slot is not usable.  The gather-skipping
 * decision above is taken at nest_route_begin: "the other slot's update is
 * still to come" means not yet issued when the route began.
 * nest_route(...) == nest_route_begin(...) + nest_route_end(ctx, slot). */
NEST_API nest_status_t nest_route_begin(nest_ctx_t* ctx, int32_t slot, const int64_t* keys,
                                        const int32_t* bag_offsets, int64_t nnz, int32_t B,
                                        const int32_t* perm, const int32_t* mb_offsets, int32_t N,
                                        void* stream);
NEST_API nest_status_t nest_route_end(nest_ctx_t* ctx, int32_t slot);

/* Dual-buffer synchronization: for every key k in both
 * the active slot's and the prefetch slot's owner key sets, copy the active
 * (already updated, written-back) row into the prefetch slot's buffer -- the
 * rows nest_route's gather skipped.  Waits inside for the active slot's update
 * and the prefetch slot's gather.  After an early push (see
 * nest_route) the same rows are re-pushed to the requesters that hold stale
 * copies.  Collective in the early-push mode: every rank calls it for the
 * same slots. */
NEST_API nest_status_t nest_dbp_refresh(nest_ctx_t* ctx, int32_t active_slot,
                               int32_t prefetch_slot, void* stream);

/* Forward of micro-batch mb: owners gather the
 * requested rows of the frozen buffer, All2All them back to the requesters
 * (on `comm`), and the source pools them per bag (sum) or expands
 * them per occurrence (pooling NONE) into out (on `compute`).
 * out: fp32 [mb_out_rows, d]; pooled row p*F+f is bag (perm[mb_off+p], f). */
NEST_API nest_status_t nest_lookup_fwd(nest_ctx_t* ctx, int32_t slot, int32_t mb, float* out,
                              void* compute, void* comm);

/* nest_lookup_fwd with bf16 output for a bf16 dense consumer: the same fp32
 * sum per bag, rounded once to bf16 (round to nearest even) when stored, so
 * out == bf16(nest_lookup_fwd's rows) bit for bit.  out: bf16 (uint16 bit
 * patterns) [mb_out_rows, d].  Pooling SUM only (else NEST_ERR_INVALID). */
NEST_API nest_status_t nest_lookup_fwd_bf16(nest_ctx_t* ctx, int32_t slot, int32_t mb, void* out,
                                            void* compute, void* comm);

/* The communication half of nest_lookup_fwd for micro-batch mb, issued early
 * (FWP stream scheduling: "communication should be launched as
 * early as possible within the frozen window"): owner send gather + embedding
 * All2All on `comm`.  The later nest_lookup_fwd of the same micro-batch then
 * only waits for it and pools on `compute`.  No-op when world == 1. */
NEST_API nest_status_t nest_lookup_prefetch(nest_ctx_t* ctx, int32_t slot, int32_t mb,
                                            void* compute, void* comm);

/* Backward of micro-batch mb: per unique
 * key of the micro-batch, deterministic segment-sum of the gradients dout of
 * the bags (pooled) or occurrences (unpooled) it occurs in, gradient All2All
 * to the owners.  After the last micro-batch (mb == N-1) every owner sums its
 * received gradients in (micro-batch, source) order and applies the
 * sparse SGD update e <- e - lr_over_B * g (Eq. 2),
 * computed from the slot buffer's frozen rows and written back to the shard
 * only (write-back): the slot buffer is not rewritten; the next slot's
 * buffer receives the written-back rows of the shared keys from
 * nest_dbp_refresh.  dout: fp32 [mb_out_rows, d] in out's layout.
 * lr_over_B = eta / |B_global|. */
NEST_API nest_status_t nest_grad_bwd_update(nest_ctx_t* ctx, int32_t slot, int32_t mb,
                                   const float* dout, float lr_over_B,
                                   void* compute, void* comm);

/* nest_grad_bwd_update for a context created with NEST_OPT_ROWWISE_ADAGRAD:
 * the same backward, and after the last micro-batch the owner applies, per
 * owner key with summed gradient G (same (micro-batch, source) order),
 *   g = grad_scale * G;  m += (1/d) sum_j g_j^2;  e -= lr * g / (sqrt(m) + eps)
 * with one fp32 accumulator m per shard row (initially 0, kept in table_mem
 * after the rows).  grad_scale = 1/|B_global|.  NEST_ERR_INVALID on an SGD
 * context (and nest_grad_bwd_update on an AdaGrad one). */
NEST_API nest_status_t nest_grad_bwd_update_adagrad(nest_ctx_t* ctx, int32_t slot, int32_t mb,
                                                    const float* dout, float grad_scale, float lr,
                                                    void* compute, void* comm);

/* Stand-in dense tower (the FWP overlap partner, not the product):
 * fixed bf16 MLP forward + backward on `stream` via cuBLAS, input = the pooled
 * rows of a micro-batch viewed as [rows/F, F*d]; writes its input gradient
 * into dout (fp32, same layout).  Requires tower_layers > 0.  dout is
 * complete when `stream` reaches it; the weight-gradient GEMMs may still run
 * on a library-internal stream (the next call, nest_join and nest_destroy
 * wait for them). */
NEST_API nest_status_t nest_tower_fwd_bwd(nest_ctx_t* ctx, const float* pooled, int64_t rows,
                                 float* dout, void* stream);

/* The same tower on bf16 pooled rows (nest_lookup_fwd_bf16), read in place
 * without the fp32 -> bf16 cast: dout is bit-identical to
 * nest_tower_fwd_bwd(pooled_fp32) whenever pooled == bf16(pooled_fp32).
 * `pooled` must stay unmodified until the deferred weight-gradient GEMMs that
 * read it finish (the next tower call, nest_join or nest_destroy). */
NEST_API nest_status_t nest_tower_fwd_bwd_bf16(nest_ctx_t* ctx, const void* pooled, int64_t rows,
                                               float* dout, void* stream);

/* Read the stand-in tower (tests): what = NEST_TOWER_WEIGHTS -> layer `layer`'s
 * weights [H, in_l] row-major (in_0 = F*d, else H) as fp32 (the fp32 master
 * copy when trained, else the bf16 weights widened); what = NEST_TOWER_TOP_GRAD
 * -> the fixed top gradient [max_batch, H] (layer ignored).  `out` is device
 * memory written on `stream` after the tower's pending work.  NEST_ERR_INVALID
 * without a tower or with a bad layer / what. */
enum { NEST_TOWER_WEIGHTS = 0, NEST_TOWER_TOP_GRAD = 1 };
NEST_API nest_status_t nest_tower_read(nest_ctx_t* ctx, int32_t what, int32_t layer, float* out, void* stream);

/* Zero-copy retrieval (also NEST_ZERO_COPY=1 at creation): batches routed
 * from now on with world == 1, one micro-batch and HBM tables skip the
 * retrieval copy (R4) -- the pool and the fused update read and update the
 * shard rows in place -- and so need no dual-buffer refresh (R5): the lookup
 * of such a batch is ordered after the previous window's update (reading
 * Q8), which is the synchronous result the refresh restores otherwise
 * (P:370-378).  Other batches keep the buffered DBP path.  Host-side only;
 * takes effect at the next nest_route_begin. */
NEST_API nest_status_t nest_set_zero_copy(nest_ctx_t* ctx, int32_t on);

/* Replace the library's internal streams with the caller's (NULL keeps
 * one): the occurrence sorts of nest_route_end and the tower's deferred dW
 * GEMMs -- e.g. streams of green contexts that split the SMs between the
 * embedding lanes and the dense tower.  The caller keeps them alive until
 * nest_destroy.  Synchronises the device first. */
NEST_API nest_status_t nest_set_streams(nest_ctx_t* ctx, void* sort_stream, void* tower_dw_stream);

/* Trained tower (tower_train = 1, NEXT-4): apply the batch's accumulated
 * dense gradient -- AllReduce over the ranks + one SGD step -- after the last
 * micro-batch's nest_tower_fwd_bwd* call (one dense update per
 * batch).  Enqueued behind the dW GEMMs on the library's dW stream, after the
 * work queued on `stream`; the next tower call waits for it.  No-op for the
 * fixed tower or when no tower call happened since the last step;
 * NEST_ERR_INVALID without a tower. */
NEST_API nest_status_t nest_tower_step(nest_ctx_t* ctx, void* stream);

/* Make `stream` wait for all work the library queued on its internal streams
 * (the tower's deferred weight-gradient GEMMs, the occurrence sorts of
 * nest_route_end).  Host-side enqueue only. */
NEST_API nest_status_t nest_join(nest_ctx_t* ctx, void* stream);

/* Host-known counts of a slot (valid after nest_route). */
NEST_API nest_status_t nest_slot_info(const nest_ctx_t* ctx, int32_t slot, nest_slot_info_t* info);

/* Device pointers to a slot's routing results (parity checks). */
NEST_API nest_status_t nest_route_view(const nest_ctx_t* ctx, int32_t slot, nest_route_view_t* view);

/* out[i] = shard row of keys[i] (device, n keys, all owned by this rank;
 * foreign / out-of-range keys give a zero row and raise the sticky error). */
NEST_API nest_status_t nest_read_rows(nest_ctx_t* ctx, const int64_t* keys, int64_t n, float* out,
                             void* stream);

/* out[i] = AdaGrad accumulator of keys[i]'s shard row (device, n keys owned by
 * this rank; NEST_ERR_INVALID on an SGD context). */
NEST_API nest_status_t nest_read_state(nest_ctx_t* ctx, const int64_t* keys, int64_t n, float* out,
                                       void* stream);

/* All2All plan of one batch, as nest_route derives it after the count
 * exchange (host-only; exposed so the multi-rank bookkeeping can be tested
 * without GPUs).  all_counts: host int32 [W][W][max_micro_batches+2]:
 * all_counts[s][o] = {keys source s sends to owner o, the same per
 * micro-batch 1..N, error flags}.  Returns the same error / capacity decision
 * nest_route takes (identical on every rank). */
typedef struct {
  int64_t uniq;                                 /* U_s of cfg->rank */
  int64_t recv;                                 /* R_o of cfg->rank */
  int64_t key_send_off[NEST_MAX_WORLD + 1];     /* key All2All send displacements */
  int64_t key_recv_off[NEST_MAX_WORLD + 1];     /* key All2All receive displacements */
  int64_t mb_uniq[NEST_MAX_MICRO_BATCHES];      /* rows received per micro-batch */
  int64_t mb_recv[NEST_MAX_MICRO_BATCHES];      /* rows sent as owner per micro-batch */
  int64_t src_base[NEST_MAX_MICRO_BATCHES + 1]; /* row base of micro-batch i (requester side) */
  int64_t own_base[NEST_MAX_MICRO_BATCHES + 1]; /* row base of micro-batch i (owner side) */
} nest_exchange_plan_t;
NEST_API nest_status_t nest_exchange_plan(const nest_config_t* cfg, int32_t N,
                                          const int32_t* all_counts, nest_exchange_plan_t* plan);

/* ---- tracing: CUDA events around every stage of the path ---- */
enum { NEST_PROFILE_STAGES = 16 };
typedef struct {
  char name[24];        /* stage: schedule, route, sort, key_a2a, owner_dedup, gather, refresh,
                           send_gather, emb_a2a, pool, tower, segsum, grad_a2a, update,
                           tower_dw (the tower's deferred weight gradients, internal stream),
                           emb_repush (early-push transport: rows the refresh re-sent) */
  int32_t stream;       /* 0 compute, 1 comm, 2 aux */
  int32_t records;      /* instrumented calls */
  int32_t launches;     /* libnest kernels launched by those calls (NCCL / cuBLAS not counted) */
  int32_t pad;
  double ms;            /* summed event-measured durations */
  double bytes;         /* summed algorithmic bytes; FLOPs for tower / tower_dw;
                           off-GPU bytes for the All2All stages */
  double units;         /* summed device-side counts: refreshed rows I (refresh),
                           owner-unique keys U_o (gather, update, owner_dedup) */
  double hbm_bytes;     /* local-HBM algorithmic bytes of the fused transport stages
                           (emb_a2a: rows gathered + rows stored locally; grad_a2a:
                           the segment-sum's reads + rows stored locally); equal to
                           `bytes` for the HBM stages, 0 for tower / tower_dw */
} nest_profile_stage_t;

typedef struct {
  double span_ms;         /* first stage start to last stage end */
  double a2a_ms;          /* summed durations of the embedding + gradient All2Alls */
  double a2a_union_ms;    /* measure of the union of those intervals */
  double a2a_exposed_ms;  /* All2All time not covered by any compute-stream stage */
  double compute_busy_ms; /* measure of the union of compute-stream stages */
  int64_t launches;       /* libnest kernels launched while tracing */
} nest_profile_summary_t;

/* on != 0: synchronize the device, drop old records and start tracing;
 * on == 0: stop tracing (records are kept for nest_profile_read). */
NEST_API nest_status_t nest_profile_enable(nest_ctx_t* ctx, int32_t on);
/* Synchronizes the device and aggregates the records: stages[NEST_PROFILE_STAGES]
 * (may be NULL) and the summary (may be NULL). */
NEST_API nest_status_t nest_profile_read(nest_ctx_t* ctx, nest_profile_stage_t* stages,
                                         nest_profile_summary_t* summary);

/* The raw stage intervals of the trace (a timeline): record i = {stage index
 * (nest_profile_stage_t order), stream kind, start ms, end ms} relative to
 * the trace start.  out: host, room for `cap` records (NULL: count only);
 * *n = the number of records (all of them, even beyond cap).  Synchronises
 * the device. */
typedef struct {
  int32_t stage, stream;
  double t0_ms, t1_ms;
} nest_profile_record_t;
NEST_API nest_status_t nest_profile_records(nest_ctx_t* ctx, nest_profile_record_t* out, int64_t cap,
                                            int64_t* n);

/* Message of the last error of ctx (or of the last failed nest_create when ctx is NULL). */
NEST_API const char* nest_last_error(const nest_ctx_t* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NEST_H_ */
