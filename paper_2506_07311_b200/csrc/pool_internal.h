// Library-internal allocator hooks (not part of the C ABI): an undo record
// for pkv_pool_prepare_append so that the batched decode step can put the
// allocator back exactly when a later stage (metadata upload, aux launch,
// attention launch) fails — the reference's all-or-nothing contract
// (pool.py:143-148, 165-169).
#pragma once
#include <cstdint>

#include "pkv200.h"

struct pkv_append_undo;

// pkv_pool_prepare_append that also returns an undo record (*undo_out, may be
// nullptr on failure).  The record must be passed to exactly one of
// pkv_pool_rollback_append / pkv_pool_release_undo before the pool is
// mutated again.
int pkv_pool_prepare_append_undo(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t* positions_out,
                                 int32_t* rows_out, uint32_t* pages_out, int64_t pages_cap,
                                 int64_t* n_pages_out, int64_t* copies_out, pkv_append_undo** undo_out);
// Restores free stack, bump counter, refcounts, tables and logical lengths;
// the mirror cells it touches are re-marked dirty.  Consumes the record.
int pkv_pool_rollback_append(pkv_pool* pool, pkv_append_undo* undo);
void pkv_pool_release_undo(pkv_append_undo* undo);

// Debug fault injection (pkv_debug_inject_failure): returns true once when
// `site` is the armed site.
bool pkv_debug_should_fail(int site);
