/*
 * pkv200 — C ABI of the B200-native paged-attention engine.
 *
 * This is the drop-in boundary for the hot path of the reference `pagedkv`
 * package (arXiv 2506.07311).  The reference is pure Python, so it has no FFI
 * of its own; every entry point below replaces one reference *Python* function
 * and is bound from Python with ctypes (INTEGRATION.md shows the binding).
 * Conventions:
 *   - every function returns a status code (PKV_OK == 0); the message of the
 *     last failure on the calling thread is available from pkv_last_error();
 *   - status codes map 1:1 onto the reference's exception classes
 *     (reference errors.py:4-41) plus Python's ValueError/IndexError where
 *     the reference raises those;
 *   - device entry points take device pointers, launch on the caller's
 *     cudaStream_t (passed as void*), never allocate and never synchronise;
 *   - the engine never owns device memory: caches, block-table mirror,
 *     workspaces and outputs belong to the caller (torch, in the Python shim).
 */
#ifndef PKV200_H
#define PKV200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum pkv_status {
  PKV_OK = 0,
  PKV_CAPACITY_EXHAUSTED = 1, /* errors.py:8  CapacityExhausted */
  PKV_DUPLICATE_SEQUENCE = 2, /* errors.py:12 DuplicateSequence */
  PKV_UNKNOWN_SEQUENCE = 3,   /* errors.py:16 UnknownSequence   */
  PKV_INVALID_PREFIX = 4,     /* errors.py:20 InvalidPrefix     */
  PKV_OUT_OF_RANGE = 5,       /* errors.py:24 OutOfRange        */
  PKV_SHAPE_MISMATCH = 6,     /* errors.py:28 ShapeMismatch     */
  PKV_NO_ALLOWED_KEYS = 7,    /* errors.py:32 NoAllowedKeys     */
  PKV_VALUE_ERROR = 8,        /* Python ValueError (pool.py:97-102, 161, 212) */
  PKV_INDEX_ERROR = 9,        /* Python IndexError (array index in pool.py:248) */
  PKV_CONFIG_ERROR = 10,      /* errors.py:40 ConfigError (unsupported shape) */
  PKV_CUDA_ERROR = 11         /* launch / device failure */
};

/* element types of caches, queries and outputs */
enum pkv_dtype { PKV_F32 = 0, PKV_F16 = 1, PKV_BF16 = 2 };

const char* pkv_last_error(void);
int pkv_abi_version(void);

/* ======================================================================
 * Page allocator — host control plane (replaces reference pool.py:88-349).
 * Bit-exact with the reference's PagePool.dump() state contract
 * (pool.py:309-329), including failed-grant free-stack reordering
 * (pool.py:143-148) and the clamped bump cursor (pool.py:286-290).
 * Internally synchronised (one mutex per pool): reserve/grow/free/fork may be
 * called from many threads as the reference contract allows (pool.py:91-94).
 * Sequences are caller-chosen int64 handles (the Python shim maps arbitrary
 * hashable ids onto handles).  Granted pages are returned to the caller, who
 * must clear them in every attached store (clear-on-grant, pool.py:122-126)
 * and perform the reported page copies (pool.py:112-120).
 * ==================================================================== */
typedef struct pkv_pool pkv_pool;

/* PagePool.__init__            pool.py:96-110 */
int pkv_pool_create(uint64_t capacity_pages, uint32_t page_size, pkv_pool** out);
void pkv_pool_destroy(pkv_pool* pool);

/* PagePool.reserve             pool.py:154-174; pages_out must hold
 * pages_for(length) entries; *n_out receives the grant size */
int pkv_pool_reserve(pkv_pool* pool, int64_t seq, int64_t length, uint32_t* pages_out,
                     int64_t* n_out);
/* PagePool.grow                pool.py:176-187 */
int pkv_pool_grow(pkv_pool* pool, int64_t seq, int64_t new_len, uint32_t* pages_out,
                  int64_t* n_out);
/* PagePool.free                pool.py:189-199 */
int pkv_pool_free(pkv_pool* pool, int64_t seq, int64_t* reclaimed_out);
/* PagePool.fork                pool.py:201-236; copy_* report the partial-page
 * copy (copy_dst == -1 when the prefix is page aligned) */
int pkv_pool_fork(pkv_pool* pool, int64_t parent, int64_t child, int64_t prefix_len,
                  int64_t* copy_src, int64_t* copy_dst, int64_t* copy_rows);
/* PagePool.privatize           pool.py:238-254; *new_page == -1 when the page
 * was already private; otherwise copy the full page old -> new */
int pkv_pool_privatize(pkv_pool* pool, int64_t seq, int64_t block_idx, int64_t* old_page,
                       int64_t* new_page);
/* KvStore.assign's copy-on-write loop (store.py:143-145): privatize the
 * given blocks in order, stopping at the first failure (earlier blocks stay
 * privatized, as with the reference's per-block loop); copies_out[2n]
 * receives the (old, new) page pairs the caller must copy in every store */
int pkv_pool_privatize_blocks(pkv_pool* pool, int64_t seq, const int64_t* blocks, int64_t n,
                              int64_t* copies_out, int64_t* n_copies_out);
/* PagePool.translate           pool.py:258-266 */
int pkv_pool_translate(pkv_pool* pool, int64_t seq, int64_t position, uint32_t* page_out,
                       uint32_t* offset_out);

/* BlockTable access            pool.py:50-71 */
int pkv_pool_has_sequence(pkv_pool* pool, int64_t seq, int32_t* out);
int pkv_pool_table_len(pkv_pool* pool, int64_t seq, int64_t* n_out);
int pkv_pool_table_entries(pkv_pool* pool, int64_t seq, uint32_t* out, int64_t cap);
int pkv_pool_table_set_entry(pkv_pool* pool, int64_t seq, int64_t idx, uint32_t value);
int pkv_pool_get_logical_len(pkv_pool* pool, int64_t seq, int64_t* out);
int pkv_pool_set_logical_len(pkv_pool* pool, int64_t seq, int64_t value);
/* sequences in insertion order (dict order of pool.py:109) */
int pkv_pool_sequence_count(pkv_pool* pool, int64_t* n_out);
int pkv_pool_sequences(pkv_pool* pool, int64_t* out, int64_t cap);

/* introspection                pool.py:272-307 */
int pkv_pool_refcount(pkv_pool* pool, uint64_t page, int64_t* out);
/* out[0..4] = capacity, live, free, never_allocated, bump_cursor */
int pkv_pool_census(pkv_pool* pool, int64_t* out5);
int pkv_pool_free_stack(pkv_pool* pool, uint32_t* out, int64_t cap, int64_t* n_out);

/* Batched decode-step planning (new; the engine's batched step API):
 * for each of n sequences append one token at position logical_len — grow the
 * table to logical_len+1 (pool.py:176-187), privatize the written block
 * (store.py:143-145) and advance logical_len (store.py:150).  All-or-nothing:
 * if the pool cannot supply every page the call fails with
 * PKV_CAPACITY_EXHAUSTED before mutating anything.  Outputs: positions_out[n],
 * rows_out[n] (mirror rows), granted pages (caller zeroes them in every store)
 * and copies_out[2n] (old,new page pairs or -1,-1; caller copies full pages). */
int pkv_pool_prepare_append(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t* positions_out,
                            int32_t* rows_out, uint32_t* pages_out, int64_t pages_cap,
                            int64_t* n_pages_out, int64_t* copies_out);

/* ---- device block-table mirror (new; SURVEY.md §7 decision 3) -----------
 * Each live table owns one row of an int32 [rows, cols] device matrix.  The
 * pool records which entries changed; the caller drains them and applies them
 * on the device with pkv_mirror_apply (or re-uploads the whole matrix after a
 * shape change, signalled by *full_resync). */
int pkv_pool_mirror_row(pkv_pool* pool, int64_t seq, int32_t* row_out);
/* One native pass of KvStore.assign's host side (store.py:117-150): scan the
 * positions (min, max, strictly increasing, contiguous run), check them
 * against the table's reserved capacity and, for strictly increasing
 * positions inside it, copy-on-write every touched block in ascending order
 * (pool.py:238-254; copies_out receives (old, fresh) page pairs for the
 * caller's page copies).  info_out[5] = {min, max, flags, pages held, mirror
 * row}; flags: PKV_ASSIGN_*.  Out-of-range or non-increasing positions
 * privatize nothing (the caller raises / dedupes first). */
#define PKV_ASSIGN_INCREASING 1
#define PKV_ASSIGN_CONTIGUOUS 2
#define PKV_ASSIGN_OUT_OF_RANGE 4
int pkv_pool_assign_prepare(pkv_pool* pool, int64_t seq, const int64_t* positions, int64_t n,
                            int64_t* info_out, int64_t* copies_out, int64_t copies_cap, int64_t* n_copies_out);

/* mutation counter of the pool: every call that can change a block table,
 * the page state or the mirror (reserve, grow, free, fork, privatize, assign
 * preparation, decode-step staging and its rollback, entry / logical-length
 * setters) bumps it.  Two equal reads bracket no such call, so a caller may
 * reuse what it derived from the tables in between (the prefill fast path of
 * paged_attention).  No reference counterpart (an engine-side memo key). */
int pkv_pool_generation(pkv_pool* pool, uint64_t* out);

/* batched table query for n sequence handles: page count and mirror row of
 * each (either output may be NULL); one call instead of two per sequence */
int pkv_pool_tables_info(pkv_pool* pool, const int64_t* seqs, int64_t n, int64_t* n_pages_out,
                         int32_t* mirror_row_out);
int pkv_pool_mirror_shape(pkv_pool* pool, int64_t* rows_out, int64_t* cols_out);
/* pairs_out holds (flat_index, value) int32 pairs; at most cap pairs */
int pkv_pool_mirror_drain(pkv_pool* pool, int32_t* pairs_out, int64_t cap, int64_t* n_out,
                          int32_t* full_resync);
int pkv_pool_mirror_pending(pkv_pool* pool, int64_t* n_out, int32_t* full_resync);
/* copy the whole host mirror (rows*cols int32) and clear the dirty state */
int pkv_pool_mirror_export(pkv_pool* pool, int32_t* out, int64_t rows, int64_t cols);

/* ======================================================================
 * Device data plane (sm_100a kernels).
 * ==================================================================== */

/* apply drained mirror pairs: table[pairs[2i]] = pairs[2i+1] */
int pkv_mirror_apply(int32_t* table, const int32_t* pairs, int64_t n_pairs, void* stream);

/* K0a  KvStore.clear_pages      store.py:95-100: zero `n` whole pages of the
 * K and V caches (page_bytes = page_size * heads * head_dim * elem_size) */
int pkv_page_zero(void* k_cache, void* v_cache, const int32_t* pages, int64_t n,
                  int64_t page_bytes, void* stream);

/* K0b  KvStore.copy_rows        store.py:85-93: for each (src, dst, rows)
 * triple copy the first `rows` rows of page src into page dst and zero the
 * rest of dst */
int pkv_page_copy(void* k_cache, void* v_cache, const int32_t* triples, int64_t n,
                  int64_t row_bytes, int32_t page_size, void* stream);
/* host -> device copy of a pinned staging buffer on `stream`, then (optional)
 * cudaEventRecord(event); and a wait for such an event (query first) — the
 * metadata staging ring of the Python shim in two calls */
int pkv_copy_h2d_record(void* dst, const void* src, int64_t bytes, void* event, void* stream);
int pkv_event_wait(void* event);
/* one copy (a fork's partial trailing page) without a metadata upload */
int pkv_page_copy1(void* k_cache, void* v_cache, int64_t src_page, int64_t dst_page, int64_t rows,
                   int64_t row_bytes, int32_t page_size, void* stream);

/* K1   KvStore.assign scatter   store.py:146-150 (reshape-and-cache):
 * cache[row(tok_row[i*row_stride], tok_pos[i])] = new[i] for K and V, where
 * row(r, p) = table[r*bt_stride + p/ps]*ps + p%ps.  Positions must be unique
 * (the shim keeps the last occurrence, reproducing numpy last-write-wins). */
int pkv_kv_append(const void* k_new, const void* v_new, int64_t n_tok, const int32_t* tok_row,
                  int32_t tok_row_stride, const int32_t* tok_pos, const int32_t* block_table,
                  int64_t bt_stride, int32_t page_size, void* k_cache, void* v_cache,
                  int64_t row_bytes, void* stream);
/* K1 for a contiguous run (the prompt of a prefill, one decode token):
 * token t goes to position pos0 + t of the sequence at mirror row seq_row; no
 * per-token metadata is uploaded (store.py:146-150 for positions
 * pos0 .. pos0 + n_tok - 1) */
int pkv_kv_append_range(const void* k_new, const void* v_new, int64_t n_tok, int32_t seq_row, int32_t pos0,
                        const int32_t* block_table, int64_t bt_stride, int32_t page_size, void* k_cache,
                        void* v_cache, int64_t row_bytes, void* stream);

/* KvStore.assign in one call (store.py:117-150) for the common case:
 * pkv_pool_assign_prepare (info_out / copies_out / n_copies_out exactly as
 * there), then — when the positions form one in-range contiguous run, no
 * block needed copy-on-write, the pool's device mirror has no pending cells
 * and block_table (that mirror, on the stream's device) is given — the K1
 * range launch and the logical-length update (max(len, last position + 1)).
 * *launched_out = 1 when it launched; 0 leaves the caller to finish the
 * assign from info_out (the preparation is never repeated). */
int pkv_kv_assign(pkv_pool* pool, int64_t seq, const int64_t* positions, int64_t n, int64_t* info_out,
                  int64_t* copies_out, int64_t copies_cap, int64_t* n_copies_out, const void* k_new,
                  const void* v_new, const int32_t* block_table, int64_t bt_stride, int32_t page_size,
                  void* k_cache, void* v_cache, int64_t row_bytes, void* stream, int32_t* launched_out);

/* K-gather: contiguous copies of paged rows — KvStore.gather / gather_view
 * (store.py:152-161, 187-190).  For view sequence s (s < n_seq) with block
 * table row seq_row[s], positions [0, cu_rows[s+1] - cu_rows[s]) land at
 * output rows cu_rows[s] .. cu_rows[s+1]-1 (cu_rows: int32 exclusive prefix,
 * n_seq + 1 entries, cu_rows[n_seq] == n_rows; device pointers).  K and V in
 * one launch; bit-exact copies.  The caller validates lengths against the
 * tables (OutOfRange) before the call. */
int pkv_kv_gather(const void* k_cache, const void* v_cache, const int32_t* block_table, int64_t bt_stride,
                  const int32_t* seq_row, const int32_t* cu_rows, int64_t n_seq, int64_t n_rows,
                  int32_t page_size, int64_t row_bytes, void* k_out, void* v_out, void* stream);

/* K2   paged_attention          attention.py:259-354 — split-K flash decode
 * over the block table with an online softmax, plus the K2c combine.
 * Query i belongs to view sequence q_seq[i] and attends keys 0..q_nkeys[i]-1
 * of that sequence (causal: q_pos+1, otherwise the sequence length; the
 * reference mask predicate attention.py:113-134 reduces to this prefix).
 * Paged mode: block_table != NULL, seq_row[s] = mirror row of view sequence s.
 * Gathered mode (gathered_attention, attention.py:357-378): block_table ==
 * NULL and seq_start[s] = first row of sequence s in contiguous K/V.
 * Query heads: hq = G * hkv; q head h reads kv head h / G.
 * Output: [n_queries, hq, head_dim] in out_dtype. */
typedef struct pkv_attention_args {
  const void* q;          /* [n_queries, hq, head_dim] */
  int32_t q_dtype;
  int64_t n_queries;
  const int32_t* q_seq;   /* [n_queries] view sequence of each query */
  const int32_t* q_nkeys; /* [n_queries] allowed key prefix of each query */
  const void* k_cache;    /* [rows, hkv, head_dim] */
  const void* v_cache;
  int32_t kv_dtype;
  const int32_t* block_table; /* paged mode: device mirror, NULL = gathered */
  int64_t bt_stride;
  const int32_t* seq_row;     /* paged mode: [n_seqs] */
  const int64_t* seq_start;   /* gathered mode: [n_seqs] */
  int32_t page_size;
  int32_t hq;
  int32_t hkv;
  int32_t head_dim;
  float scale;
  void* out;
  int32_t out_dtype;
  void* workspace; /* pkv_attention_workspace_bytes() bytes, 256-B aligned */
  int64_t workspace_bytes;
  int32_t num_sms;  /* 0 = query the device */
  int32_t target_waves; /* 0 = default work-splitting heuristic */
  void* prof_start; /* optional cudaEvent_t recorded right before the K2 launch */
  void* prof_stop;  /* optional cudaEvent_t recorded right after the K2 launch */
  /* kernel selection: 0 = auto (bf16 caches -> tensor-core K2, fp32/fp16 ->
   * fp32 CUDA-core K2, which keeps the reference's 1e-5 bar), 1 = force the
   * fp32 CUDA-core kernel, 2 = force the tensor-core kernel */
  int32_t mode;
  /* optional fused append (decode step, one query per sequence): the token at
   * position q_nkeys[i]-1 of query i's sequence is taken from k_new/v_new
   * [n_queries, hkv, head_dim] and written into its page first */
  const void* k_new;
  const void* v_new;
  /* tensor-core path only: the work plan from pkv_attention_plan(), both the
   * host copy (read by the launcher) and an identical device copy */
  const int32_t* plan;
  const int32_t* plan_host;
  /* optional: copy meta_bytes from pinned meta_host to meta_dev on the stream
   * before the launch (the packed [q_seq | nkeys | rows | plan] block the
   * device pointers above point into) */
  const void* meta_host;
  void* meta_dev;
  int64_t meta_bytes;
} pkv_attention_args;

/* Host planner of the tensor-core decode (a serving scheduler's job: the
 * per-query key counts are host metadata).  q_row[i] is the mirror row of
 * query i's sequence (paged) or its first K/V row (gathered).  Chooses the
 * head blocking, even page splits, a size-sorted item order and a greedy
 * LPT assignment of items to CTAs; writes at most
 * pkv_attention_plan_ints(n_queries, hq) int32 into plan_out (*n_out = used).
 * num_sms <= 0 queries the device; target_waves <= 0 uses the default. */
int64_t pkv_attention_plan_ints(int64_t n_queries, int32_t hq);
int pkv_attention_plan(const int32_t* q_nkeys, const int32_t* q_row, int64_t n_queries,
                       int32_t page_size, int32_t hq, int32_t hkv, int32_t num_sms,
                       int32_t target_waves, int32_t* plan_out, int64_t cap, int64_t* n_out);
/* the same with the head dim the planner's byte costs use (pkv_attention_plan
 * assumes 128; the batched decode step derives it from the store rows) */
int pkv_attention_plan_d(const int32_t* q_nkeys, const int32_t* q_row, int64_t n_queries,
                         int32_t page_size, int32_t hq, int32_t hkv, int32_t head_dim, int32_t num_sms,
                         int32_t target_waves, int32_t* plan_out, int64_t cap, int64_t* n_out);

/* One decode step's host work for n sequences of a pool — the batched form of
 * DecodeSession.step (decoder.py:263-284): pkv_pool_prepare_append (grow,
 * copy-on-write, logical_len += 1), then the packed metadata
 * [q_seq | nkeys | rows | plan] written into meta (pinned host memory,
 * meta_cap int32; *meta_used receives the count).  The caller clears the
 * granted pages / performs the reported copies in every store, uploads the
 * metadata (or passes it as meta_host to pkv_paged_attention) and launches. */
int pkv_decode_step_prepare(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t page_size,
                            int32_t hq, int32_t hkv, int32_t* meta, int64_t meta_cap,
                            int64_t* meta_used, uint32_t* pages_out, int64_t pages_cap,
                            int64_t* n_pages_out, int64_t* copies_out);

/* The whole host half of a batched decode step in one call (the serving-loop
 * form of DecodeSession.step, decoder.py:263-284): waits for the staging
 * slot, runs pkv_decode_step_prepare into meta_host, appends the granted
 * pages, copy-on-write triples and dirty mirror pairs, uploads everything
 * with one cudaMemcpyAsync to meta_dev (recording slot_event), then launches
 * the page clears / copies in every attached store (clear-on-grant,
 * pool.py:122-126; copy-on-write, store.py:143-145) and the mirror update.
 * If the device mirror's shape changed (or it is absent) needs_resync is set:
 * the caller re-exports the mirror before launching attention.  The
 * attention metadata (meta_used int32) sits at the start of meta_dev. */
typedef struct pkv_step_stage_args {
  pkv_pool* pool;
  const int64_t* seqs;
  int64_t n;
  int32_t page_size;
  int32_t hq;
  int32_t hkv;
  int32_t* meta_host;   /* pinned */
  int32_t* meta_dev;
  int64_t meta_cap;     /* int32 entries of both slots */
  void* slot_event;     /* cudaEvent_t or NULL */
  int32_t n_stores;
  void* const* k_caches;
  void* const* v_caches;
  int64_t row_bytes;
  int32_t* mirror_dev;
  int64_t mirror_rows;
  int64_t mirror_cols;
  int64_t meta_used;    /* out */
  int32_t needs_resync; /* out */
  int32_t launches;     /* out */
  int64_t n_granted;    /* out: granted pages at meta_host[granted_off ...] */
  int64_t granted_off;
  int64_t n_copies;     /* out: (src, dst, rows) triples at meta_host[copies_off ...] */
  int64_t copies_off;
} pkv_step_stage_args;
int64_t pkv_decode_step_stage_ints(int64_t n, int32_t hq);
int pkv_decode_step_stage(pkv_step_stage_args* args, void* stream);

/* Workspace bound: the split planner never creates more than
 * n_queries + 8192 key splits, so the bound depends only on the query count. */
/* pkv_decode_step computes the NEXT step's plan (every key count + 1) while
 * the GPU runs the current one and memoises it per host thread;
 * pkv_attention_plan returns the memoised plan when its inputs match exactly
 * (the plan is a pure function of them).  Reset drops the memo (tests). */
void pkv_plan_memo_reset(void);

int64_t pkv_attention_workspace_bytes(int64_t n_queries, int32_t hq, int32_t head_dim);
int pkv_paged_attention(const pkv_attention_args* args, void* stream);

/* One whole decode token step in one call — the serving-loop form of
 * DecodeSession.step (decoder.py:263-284) for a batch, and the entry a
 * foreign binding drives with HOST buffers:
 *   [H2D q / k_new / v_new from q_host / k_host / v_host (each optional)]
 *   -> pkv_decode_step_stage(stage) -> pkv_paged_attention(attn, K1 fused)
 *   -> [D2H of attn->out into out_host (optional)]
 * all on `stream`.  attn->q / k_new / v_new / out are the DEVICE buffers the
 * copies land in / read from; attn's metadata pointers (q_seq, q_nkeys,
 * seq_row, plan, plan_host, n_queries) are filled here from the stage slot.
 * Page work needs the stores attached (stage->n_stores > 0).  When the
 * allocator changed the block-table shape (stage->needs_resync) nothing is
 * launched after the stage and io->launched = 0: attn's metadata pointers are
 * filled, the caller re-exports the mirror, sets attn->block_table /
 * bt_stride and launches pkv_paged_attention(attn) itself.  Host buffers should be
 * pinned for the copies to be asynchronous.  attn->out may itself be mapped
 * pinned host memory (cudaHostAlloc under UVA): the kernel then stores the
 * result straight to the host and out_host stays NULL (the Python shim does
 * this for pinned outputs; no trailing D2H on the critical path). */
typedef struct pkv_decode_io {
  const void* q_host;   /* NULL: attn->q already holds the queries */
  const void* k_host;
  const void* v_host;
  void* out_host;       /* NULL: leave the output on the device */
  int64_t q_bytes;
  int64_t kv_bytes;     /* each of k and v */
  int64_t out_bytes;
  int32_t launched;     /* out: 1 = attention launched (and D2H issued) */
  int32_t launches;     /* out: kernels launched by this call */
} pkv_decode_io;
int pkv_decode_step(pkv_step_stage_args* stage, pkv_attention_args* attn, pkv_decode_io* io, void* stream);

/* CUDA-graph mode of the same step: identical host work and semantics, but
 * the step's device work (input copies, metadata copy, page / mirror aux
 * kernel, fused append + decode) is recorded and replayed as ONE
 * cudaGraphLaunch from a cache of executable graphs (one per topology; only
 * the changed parameters are updated between launches).  Steps with a host
 * `out_host` copy or on the fp32 path run as pkv_decode_step.  Replaces the
 * per-token launch sequence of DecodeSession.step (decoder.py:263-284). */
typedef struct pkv_step_graph pkv_step_graph;
int pkv_step_graph_create(pkv_step_graph** out);
void pkv_step_graph_destroy(pkv_step_graph* graphs);
int pkv_step_graph_stats(pkv_step_graph* graphs, int64_t* launches, int64_t* builds);
int pkv_decode_step_graph(pkv_step_graph* graphs, pkv_step_stage_args* stage, pkv_attention_args* attn,
                          pkv_decode_io* io, void* stream);

/* K3   causal / suffix prefill on tcgen05 tensor cores (16-bit caches).
 * Replaces _streaming_attention (attention.py:259-329) under the
 * self-attention and suffix metas (attention.py:81-84, 98-110): the queries
 * of view sequence s are the q_len[s] consecutive positions ending at
 * seq_len[s]-1, stored contiguously from row q_start[s] of q.  The host
 * planner cuts them into work items (one kv head x 128/G query positions,
 * longest first); the caller uploads the plan and passes both copies. */
typedef struct pkv_prefill_args {
  const void* q;             /* [total_q, hq, head_dim], same dtype as the cache */
  int64_t total_q;
  const void* k_cache;       /* [cache_rows, hkv, head_dim] */
  const void* v_cache;
  int32_t kv_dtype;          /* PKV_BF16 or PKV_F16 */
  int64_t cache_rows;
  const int32_t* block_table; /* device mirror */
  int64_t bt_stride;
  int32_t page_size;         /* power of two >= 8 */
  int32_t hq;
  int32_t hkv;
  int32_t head_dim;          /* 64 or 128 */
  float scale;
  int32_t causal;
  void* out;                 /* [total_q, hq, head_dim], fp32 or the cache dtype */
  int32_t out_dtype;
  const int32_t* plan;       /* device copy of the pkv_prefill_plan() items */
  int64_t n_items;
  void* prof_start;          /* optional cudaEvent_t pair around the launch */
  void* prof_stop;
  void* debug;               /* optional device uint64[512]: timeline of CTA 0 (NULL = off) */
} pkv_prefill_args;

int pkv_prefill_supported(int32_t hq, int32_t hkv, int32_t head_dim, int32_t page_size,
                          int32_t kv_dtype);
/* int32 entries the plan of these sequences needs (8 per work item) */
int64_t pkv_prefill_plan_ints(const int32_t* q_len, int64_t n_seqs, int32_t hq, int32_t hkv);
/* host planner: q_start (int64), q_len, seq_len, seq_row per view sequence */
int pkv_prefill_plan(const int64_t* q_start, const int32_t* q_len, const int32_t* seq_len,
                     const int32_t* seq_row, int64_t n_seqs, int32_t hq, int32_t hkv,
                     int32_t causal, int32_t* plan_out, int64_t cap, int64_t* n_items_out);
/* The K3 route of paged_attention in one host pass (attention.py:81-84,
 * 98-110, 332-354): q_seq / q_pos (int64, q_seq non-decreasing), seq_len
 * (int64) and seq_row per view sequence.  Suffix-shaped metadata (each
 * sequence's queries one run of consecutive positions ending at its last
 * key): *n_items_out >= 0, *max_run_out = longest run and, when build > 0 and
 * the longest run is at least build positions, the memoised plan in plan_out
 * (else *n_items_out = 0).  Otherwise *n_items_out = -1.
 * *generation_out names the memoised plan: the same value on the same host
 * thread means the same plan (a caller may reuse its device copy). */
int pkv_prefill_plan_meta(const int64_t* q_seq, const int64_t* q_pos, int64_t n_q, const int64_t* seq_len,
                          const int32_t* seq_row, int64_t n_seqs, int32_t hq, int32_t hkv, int32_t causal,
                          int32_t build, int32_t* plan_out, int64_t cap, int64_t* n_items_out,
                          int64_t* max_run_out, int64_t* generation_out);
int pkv_paged_prefill(const pkv_prefill_args* args, void* stream);

/* number of SMs of the current device (0 when no device is visible) */
int pkv_device_sm_count(int32_t* out);

/* Debug: per-CTA globaltimer timeline of the tensor-core decode kernel
 * (64 stamps per CTA).  enable = 1/0 switches recording on/off and clears the
 * buffer (-1 leaves it); out (n entries, may be NULL) receives the stamps.
 * Synchronous. */
int pkv_debug_trace(int32_t enable, uint64_t* out, int64_t n);

/* Debug: make the next decode step fail at `site` (one shot; 0 disarms):
 * PKV_FAIL_STEP_UPLOAD = the metadata upload of pkv_decode_step_stage,
 * PKV_FAIL_STEP_LAUNCH = the attention launch of pkv_decode_step.  The step
 * returns PKV_CUDA_ERROR and the allocator is rolled back (tests of the
 * all-or-nothing contract, pool.py:143-148, 165-169). */
/* Debug: host phase stamps (ns since entry) of this thread's last
 * pkv_decode_step: [1] input copies issued, [2] staging slot free, [3]
 * allocator + plan, [4] side blocks, [5] metadata upload issued, [6] aux
 * kernel issued, [7] before / [8] after the decode launch, [9] output copy
 * issued, [10] next plan speculated; [11] the entry time itself (steady clock,
 * ns since its epoch: CLOCK_MONOTONIC on Linux). */
int pkv_debug_step_times(int64_t* out, int32_t n);

#define PKV_FAIL_STEP_UPLOAD 1
#define PKV_FAIL_STEP_LAUNCH 2
int pkv_debug_inject_failure(int32_t site);

#ifdef __cplusplus
}
#endif
#endif /* PKV200_H */
