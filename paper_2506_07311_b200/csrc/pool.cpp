// Host page allocator with a device block-table mirror.
//
// Replaces the reference PagePool (pkg/src/pagedkv/pool.py:88-349) behind the
// C ABI of include/pkv200.h.  The observable state — free stack order, clamped
// bump cursor, refcount census, tables — follows the reference exactly,
// including the failure-path quirks SURVEY.md Appendix A documents, so that
// PagePool.dump() of the Python shim is bit-identical to the reference's.
//
// What is new relative to the reference: every table owns a row of an int32
// mirror matrix that the data-plane kernels read (K1 append, K2 attention,
// K3 prefill).  Mutations record dirty (row, col) cells; the shim drains them
// and applies them on the device with one tiny kernel, so a decode step that
// grows B tables uploads B integers instead of the whole table.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "pkv200.h"
#include "status.h"
#include "pool_internal.h"

namespace {

struct Table {
  std::vector<uint32_t> entries;
  int64_t logical_len = 0;
  int32_t mirror_row = -1;
  uint64_t order = 0;  // insertion order (dict order of pool.py:109)
};

// Python's floor division for a positive divisor.
inline int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

}  // namespace

struct pkv_pool {
  std::mutex mu;
  // bumped by every entry point that can change a table, the page state or
  // the mirror's contents: equal values across two reads mean no such call
  // ran in between (the attention entry points' memo check)
  std::atomic<uint64_t> generation{0};
  uint64_t capacity = 0;
  uint32_t page_size = 0;
  std::vector<uint32_t> free_stack;  // back() is the top (deque.pop())
  uint64_t bump_raw = 0;             // itertools.count value (may overshoot)
  std::vector<int64_t> refcount;     // grown on demand, logically [capacity]
  int64_t nonzero = 0;               // count_nonzero(refcount)
  int64_t shared = 0;                // pages with refcount > 1 (0: no copy-on-write anywhere)
  std::unordered_map<int64_t, Table> tables;
  uint64_t next_order = 0;

  // device mirror (host copy + dirty cells)
  int64_t mrows = 0, mcols = 0;
  std::vector<int32_t> mirror;
  std::vector<int32_t> free_rows;
  int32_t next_row = 0;
  std::vector<int64_t> dirty;
  bool full_resync = true;

  int64_t pages_for(int64_t length) const { return -floordiv(-length, page_size); }
  uint64_t bump_cursor() const { return std::min<uint64_t>(bump_raw, capacity); }

  int64_t ref(uint64_t page) const { return page < refcount.size() ? refcount[page] : 0; }
  void set_ref(uint64_t page, int64_t v) {
    if (page >= refcount.size()) refcount.resize(std::max<uint64_t>(page + 1, refcount.size() * 2), 0);
    int64_t old = refcount[page];
    refcount[page] = v;
    nonzero += (v != 0) - (old != 0);
    shared += (v > 1) - (old > 1);
  }

  // pool.py:130-136
  bool take_one(uint32_t* page) {
    if (!free_stack.empty()) {
      *page = free_stack.back();
      free_stack.pop_back();
      return true;
    }
    uint64_t p = bump_raw++;
    if (p < capacity) {
      *page = static_cast<uint32_t>(p);
      return true;
    }
    return false;
  }

  // pool.py:138-150: on shortfall the pages taken so far are pushed back in
  // taken order (deque.extend), which can reverse the stack.
  bool take(int64_t count, std::vector<uint32_t>* got) {
    got->clear();
    for (int64_t i = 0; i < count; ++i) {
      uint32_t p;
      if (!take_one(&p)) {
        free_stack.insert(free_stack.end(), got->begin(), got->end());
        got->clear();
        return false;
      }
      got->push_back(p);
    }
    return true;
  }

  // pool.py:339-349 — table order; IndexError (numpy) beyond capacity
  int release(const std::vector<uint32_t>& pages, int64_t* reclaimed) {
    int64_t n = 0;
    for (uint32_t p : pages) {
      if (p >= capacity) {
        *reclaimed = n;
        return pkv::fail(PKV_INDEX_ERROR, "index %u is out of bounds for refcounts", p);
      }
      int64_t v = ref(p) - 1;
      set_ref(p, v);
      if (v == 0) {
        free_stack.push_back(p);
        ++n;
      }
    }
    *reclaimed = n;
    return PKV_OK;
  }

  Table* find(int64_t seq) {
    auto it = tables.find(seq);
    return it == tables.end() ? nullptr : &it->second;
  }

  // ---- mirror bookkeeping ---------------------------------------------
  void ensure_shape(int64_t rows, int64_t cols) {
    if (rows <= mrows && cols <= mcols) return;
    int64_t nr = std::max<int64_t>(mrows, 1), nc = std::max<int64_t>(mcols, 1);
    while (nr < rows) nr *= 2;
    while (nc < cols) nc *= 2;
    std::vector<int32_t> m(static_cast<size_t>(nr * nc), 0);
    for (int64_t r = 0; r < mrows; ++r)
      std::memcpy(&m[r * nc], &mirror[r * mcols], sizeof(int32_t) * mcols);
    mirror.swap(m);
    mrows = nr;
    mcols = nc;
    full_resync = true;
    dirty.clear();
  }
  int32_t alloc_row() {
    int32_t r;
    if (!free_rows.empty()) {
      r = free_rows.back();
      free_rows.pop_back();
    } else {
      r = next_row++;
    }
    ensure_shape(r + 1, mcols);
    return r;
  }
  void mark(const Table& t, int64_t col) {
    ensure_shape(t.mirror_row + 1, col + 1);
    int64_t flat = t.mirror_row * mcols + col;
    mirror[flat] = static_cast<int32_t>(t.entries[col]);
    if (!full_resync) dirty.push_back(flat);
  }
  void append_entries(Table& t, const std::vector<uint32_t>& pages) {
    int64_t start = static_cast<int64_t>(t.entries.size());
    t.entries.insert(t.entries.end(), pages.begin(), pages.end());
    if (!t.entries.empty()) ensure_shape(t.mirror_row + 1, static_cast<int64_t>(t.entries.size()));
    for (int64_t c = start; c < static_cast<int64_t>(t.entries.size()); ++c) mark(t, c);
  }
  Table& insert(int64_t seq) {
    Table& t = tables[seq];
    t.order = next_order++;
    t.mirror_row = alloc_row();
    return t;
  }
  void erase(int64_t seq) {
    auto it = tables.find(seq);
    if (it == tables.end()) return;
    free_rows.push_back(it->second.mirror_row);
    tables.erase(it);
  }
};

namespace {

void copy_out(const std::vector<uint32_t>& v, uint32_t* out, int64_t* n) {
  if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
  if (n) *n = static_cast<int64_t>(v.size());
}

#define LOCK(p)                                                        \
  if (!(p)) return pkv::fail(PKV_VALUE_ERROR, "null pool handle");     \
  std::lock_guard<std::mutex> _guard((p)->mu)

// LOCK for the mutating entry points
#define LOCK_MUT(p) \
  LOCK(p);          \
  (p)->generation.fetch_add(1, std::memory_order_relaxed)

#define TABLE_OR_FAIL(t, p, seq)                                                      \
  Table* t = (p)->find(seq);                                                          \
  if (!t) return pkv::fail(PKV_UNKNOWN_SEQUENCE, "no block table for sequence %lld", \
                           static_cast<long long>(seq))

}  // namespace

// copy-on-write of one block of a table (pool.py:238-254), pool lock held
static int privatize_locked(pkv_pool* pool, Table* t, int64_t block_idx, int64_t* old_page, int64_t* new_page) {
  const int64_t n = static_cast<int64_t>(t->entries.size());
  int64_t idx = block_idx < 0 ? block_idx + n : block_idx;
  if (idx < 0 || idx >= n) return pkv::fail(PKV_INDEX_ERROR, "array index out of range");
  uint32_t old = t->entries[idx];
  if (old >= pool->capacity)
    return pkv::fail(PKV_INDEX_ERROR, "index %u is out of bounds for refcounts", old);
  if (old_page) *old_page = old;
  if (pool->ref(old) <= 1) return PKV_OK;
  std::vector<uint32_t> got;
  if (!pool->take(1, &got))
    return pkv::fail(PKV_CAPACITY_EXHAUSTED, "pool cannot supply 1 pages (%zu free, bump at %llu/%llu)",
                     pool->free_stack.size(), static_cast<unsigned long long>(pool->bump_cursor()),
                     static_cast<unsigned long long>(pool->capacity));
  uint32_t fresh = got[0];
  pool->set_ref(fresh, 1);
  t->entries[idx] = fresh;
  pool->mark(*t, idx);
  if (new_page) *new_page = fresh;
  int64_t dummy;
  return pool->release(std::vector<uint32_t>{old}, &dummy);
}

extern "C" {

int pkv_pool_create(uint64_t capacity_pages, uint32_t page_size, pkv_pool** out) {
  if (!out) return pkv::fail(PKV_VALUE_ERROR, "null out pointer");
  *out = nullptr;
  if (capacity_pages == 0 || capacity_pages > (uint64_t(1) << 32))
    return pkv::fail(PKV_VALUE_ERROR, "capacity_pages must be in [1, 2^32], got %llu",
                     static_cast<unsigned long long>(capacity_pages));
  if (page_size == 0 || (page_size & (page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a positive power of two, got %u",
                     page_size);
  auto* p = new pkv_pool();
  p->capacity = capacity_pages;
  p->page_size = page_size;
  *out = p;
  return PKV_OK;
}

void pkv_pool_destroy(pkv_pool* pool) { delete pool; }

int pkv_pool_reserve(pkv_pool* pool, int64_t seq, int64_t length, uint32_t* pages_out,
                     int64_t* n_out) {
  LOCK_MUT(pool);
  if (n_out) *n_out = 0;
  if (length < 0) return pkv::fail(PKV_VALUE_ERROR, "length must be non-negative, got %lld",
                                   static_cast<long long>(length));
  if (pool->find(seq))
    return pkv::fail(PKV_DUPLICATE_SEQUENCE, "sequence %lld already has a block table",
                     static_cast<long long>(seq));
  Table& t = pool->insert(seq);
  std::vector<uint32_t> got;
  if (!pool->take(pool->pages_for(length), &got)) {
    pool->erase(seq);
    return pkv::fail(PKV_CAPACITY_EXHAUSTED, "pool cannot supply %lld pages (%zu free, bump at %llu/%llu)",
                     static_cast<long long>(pool->pages_for(length)), pool->free_stack.size(),
                     static_cast<unsigned long long>(pool->bump_cursor()),
                     static_cast<unsigned long long>(pool->capacity));
  }
  for (uint32_t p : got) pool->set_ref(p, 1);
  pool->append_entries(t, got);
  copy_out(got, pages_out, n_out);
  return PKV_OK;
}

int pkv_pool_grow(pkv_pool* pool, int64_t seq, int64_t new_len, uint32_t* pages_out,
                  int64_t* n_out) {
  LOCK_MUT(pool);
  if (n_out) *n_out = 0;
  TABLE_OR_FAIL(t, pool, seq);
  int64_t needed = pool->pages_for(new_len) - static_cast<int64_t>(t->entries.size());
  if (needed <= 0) return PKV_OK;
  std::vector<uint32_t> got;
  if (!pool->take(needed, &got))
    return pkv::fail(PKV_CAPACITY_EXHAUSTED, "pool cannot supply %lld pages (%zu free, bump at %llu/%llu)",
                     static_cast<long long>(needed), pool->free_stack.size(),
                     static_cast<unsigned long long>(pool->bump_cursor()),
                     static_cast<unsigned long long>(pool->capacity));
  for (uint32_t p : got) pool->set_ref(p, 1);
  pool->append_entries(*t, got);
  copy_out(got, pages_out, n_out);
  return PKV_OK;
}

int pkv_pool_free(pkv_pool* pool, int64_t seq, int64_t* reclaimed_out) {
  LOCK_MUT(pool);
  if (reclaimed_out) *reclaimed_out = 0;
  TABLE_OR_FAIL(t, pool, seq);
  std::vector<uint32_t> pages = std::move(t->entries);
  pool->erase(seq);
  int64_t n = 0;
  int st = pool->release(pages, &n);
  if (reclaimed_out) *reclaimed_out = n;
  return st;
}

int pkv_pool_fork(pkv_pool* pool, int64_t parent, int64_t child, int64_t prefix_len,
                  int64_t* copy_src, int64_t* copy_dst, int64_t* copy_rows) {
  LOCK_MUT(pool);
  if (copy_src) *copy_src = -1;
  if (copy_dst) *copy_dst = -1;
  if (copy_rows) *copy_rows = 0;
  TABLE_OR_FAIL(pt, pool, parent);
  if (prefix_len < 0) return pkv::fail(PKV_VALUE_ERROR, "prefix_len must be non-negative, got %lld",
                                       static_cast<long long>(prefix_len));
  if (prefix_len > pt->logical_len)
    return pkv::fail(PKV_INVALID_PREFIX, "prefix %lld exceeds parent length %lld",
                     static_cast<long long>(prefix_len), static_cast<long long>(pt->logical_len));
  if (pool->find(child))
    return pkv::fail(PKV_DUPLICATE_SEQUENCE, "sequence %lld already has a block table",
                     static_cast<long long>(child));
  // pointers into the unordered_map stay valid across insertions
  Table& ct = pool->insert(child);
  pt = pool->find(parent);
  const int64_t ps = pool->page_size;
  const int64_t full = prefix_len / ps, rem = prefix_len % ps;
  bool have_copy = false;
  uint32_t cpage = 0;
  if (rem) {
    std::vector<uint32_t> got;
    if (!pool->take(1, &got)) {
      pool->erase(child);
      return pkv::fail(PKV_CAPACITY_EXHAUSTED, "pool cannot supply 1 pages (%zu free, bump at %llu/%llu)",
                       pool->free_stack.size(), static_cast<unsigned long long>(pool->bump_cursor()),
                       static_cast<unsigned long long>(pool->capacity));
    }
    have_copy = true;
    cpage = got[0];
  }
  // parent.entries[:full] — Python slicing truncates silently
  int64_t n_shared = std::min<int64_t>(full, static_cast<int64_t>(pt->entries.size()));
  std::vector<uint32_t> shared(pt->entries.begin(), pt->entries.begin() + n_shared);
  for (uint32_t p : shared) {
    if (p >= pool->capacity)
      return pkv::fail(PKV_INDEX_ERROR, "index %u is out of bounds for refcounts", p);
    pool->set_ref(p, pool->ref(p) + 1);
  }
  pool->append_entries(ct, shared);
  if (have_copy) {
    pool->set_ref(cpage, 1);
    if (full >= static_cast<int64_t>(pt->entries.size()))
      return pkv::fail(PKV_INDEX_ERROR, "array index out of range");
    if (copy_src) *copy_src = pt->entries[full];
    if (copy_dst) *copy_dst = cpage;
    if (copy_rows) *copy_rows = rem;
    pool->append_entries(ct, std::vector<uint32_t>{cpage});
  }
  ct.logical_len = prefix_len;
  return PKV_OK;
}

int pkv_pool_privatize(pkv_pool* pool, int64_t seq, int64_t block_idx, int64_t* old_page,
                       int64_t* new_page) {
  LOCK_MUT(pool);
  if (old_page) *old_page = -1;
  if (new_page) *new_page = -1;
  TABLE_OR_FAIL(t, pool, seq);
  return privatize_locked(pool, t, block_idx, old_page, new_page);
}

int pkv_pool_privatize_blocks(pkv_pool* pool, int64_t seq, const int64_t* blocks, int64_t n,
                              int64_t* copies_out, int64_t* n_copies_out) {
  *n_copies_out = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t old = -1, fresh = -1;
    const int st = pkv_pool_privatize(pool, seq, blocks[i], &old, &fresh);
    if (st) return st;  // earlier blocks stay privatized, as with the reference's loop
    if (fresh >= 0) {
      copies_out[2 * *n_copies_out] = old;
      copies_out[2 * *n_copies_out + 1] = fresh;
      ++*n_copies_out;
    }
  }
  return PKV_OK;
}

int pkv_pool_assign_prepare(pkv_pool* pool, int64_t seq, const int64_t* positions, int64_t n,
                            int64_t* info_out, int64_t* copies_out, int64_t copies_cap, int64_t* n_copies_out) {
  if (n < 0 || (n > 0 && !positions) || !info_out || !n_copies_out)
    return pkv::fail(PKV_VALUE_ERROR, "bad assign inputs");
  *n_copies_out = 0;
  // the common case first: a contiguous run p0, p0+1, ... (a prompt, a
  // decode token) is one vectorised xor/or pass; anything else gets the
  // min / max / non-increasing-step scan
  const int64_t p0 = n ? positions[0] : 0;
  uint64_t diff = 0;
  for (int64_t i = 0; i < n; ++i) diff |= static_cast<uint64_t>(positions[i] ^ (p0 + i));
  int64_t lo = p0, hi = n ? p0 + n - 1 : p0, steps_down = 0;
  if (diff) {
    hi = p0;
    for (int64_t i = 1; i < n; ++i) {
      const int64_t x = positions[i];
      steps_down += x <= positions[i - 1];
      lo = std::min(lo, x);
      hi = std::max(hi, x);
    }
  }
  const bool increasing = steps_down == 0;
  LOCK(pool);  // a read unless it privatizes blocks below
  TABLE_OR_FAIL(t, pool, seq);
  const int64_t ps = static_cast<int64_t>(pool->page_size);
  const int64_t n_pages = static_cast<int64_t>(t->entries.size());
  int64_t flags = 0;
  if (increasing) flags |= PKV_ASSIGN_INCREASING;
  if (increasing && hi - lo == n - 1) flags |= PKV_ASSIGN_CONTIGUOUS;
  const bool in_range = n == 0 || (lo >= 0 && hi < n_pages * ps);
  if (!in_range) flags |= PKV_ASSIGN_OUT_OF_RANGE;
  info_out[0] = lo;
  info_out[1] = hi;
  info_out[2] = flags;
  info_out[3] = n_pages;
  info_out[4] = t->mirror_row;
  // no page of the pool is shared: nothing to copy-on-write
  if (!in_range || !increasing || n == 0 || pool->shared == 0) return PKV_OK;
  pool->generation.fetch_add(1, std::memory_order_relaxed);
  // touched blocks, ascending and distinct (the positions increase): a
  // contiguous run walks its block range, otherwise every position's block
  // (a shift for the power-of-two page sizes: no per-position division)
  const bool pow2 = (ps & (ps - 1)) == 0;
  const int shift = pow2 ? __builtin_ctzll(static_cast<unsigned long long>(ps)) : 0;
  const bool contiguous = (flags & PKV_ASSIGN_CONTIGUOUS) != 0;
  const int64_t n_iter = contiguous ? (hi / ps - lo / ps + 1) : n;
  int64_t prev = -1;
  for (int64_t i = 0; i < n_iter; ++i) {
    const int64_t b = contiguous ? lo / ps + i : (pow2 ? positions[i] >> shift : positions[i] / ps);
    if (b == prev) continue;
    prev = b;
    int64_t old = -1, fresh = -1;
    const int st = privatize_locked(pool, t, b, &old, &fresh);
    if (st) return st;  // earlier blocks stay privatized, as with the reference's loop
    if (fresh >= 0) {
      if (2 * *n_copies_out + 2 > copies_cap) return pkv::fail(PKV_VALUE_ERROR, "copy buffer too small");
      copies_out[2 * *n_copies_out] = old;
      copies_out[2 * *n_copies_out + 1] = fresh;
      ++*n_copies_out;
    }
  }
  return PKV_OK;
}

int pkv_pool_prepare_append(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t* positions_out,
                            int32_t* rows_out, uint32_t* pages_out, int64_t pages_cap,
                            int64_t* n_pages_out, int64_t* copies_out) {
  return pkv_pool_prepare_append_undo(pool, seqs, n, positions_out, rows_out, pages_out, pages_cap,
                                      n_pages_out, copies_out, nullptr);
}

}  // extern "C"

// Undo record of one pkv_pool_prepare_append: everything phase 2 changed.
// Phase 2 only pops the free stack / bumps (CoW releases never reach a zero
// refcount), so restoring the popped tail and the raw bump counter puts the
// free list back bit-exactly.
struct pkv_append_undo {
  std::vector<uint32_t> stack_tail;  // the free-stack tail phase 2 could pop
  size_t stack_size = 0;
  uint64_t bump_raw = 0;
  struct Seq {
    int64_t handle;
    int64_t logical_len;
    size_t n_entries;
    int64_t cow_block;  // -1: no copy-on-write
    uint32_t cow_old;
  };
  std::vector<Seq> seqs;
  std::vector<uint32_t> granted;  // refcount 0 -> 1
};

int pkv_pool_prepare_append_undo(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t* positions_out,
                                 int32_t* rows_out, uint32_t* pages_out, int64_t pages_cap,
                                 int64_t* n_pages_out, int64_t* copies_out, pkv_append_undo** undo_out) {
  if (undo_out) *undo_out = nullptr;
  LOCK_MUT(pool);
  *n_pages_out = 0;
  const int64_t ps = pool->page_size;
  // phase 1: validate and count pages without mutating
  std::vector<Table*> tabs(n);
  int64_t need = 0;
  for (int64_t i = 0; i < n; ++i) {
    Table* t = pool->find(seqs[i]);
    if (!t) return pkv::fail(PKV_UNKNOWN_SEQUENCE, "no block table for sequence %lld",
                             static_cast<long long>(seqs[i]));
    tabs[i] = t;
  }
  {  // a sequence may appear once per step (O(n log n) check)
    std::vector<Table*> sorted(tabs);
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
      return pkv::fail(PKV_VALUE_ERROR, "a sequence is listed twice in one decode step");
  }
  for (int64_t i = 0; i < n; ++i) {
    Table* t = tabs[i];
    const int64_t pos = t->logical_len;
    if (pos < 0 || pos >= (int64_t(1) << 31) - 1)
      return pkv::fail(PKV_OUT_OF_RANGE, "position %lld not addressable", static_cast<long long>(pos));
    const int64_t grow = pool->pages_for(pos + 1) - static_cast<int64_t>(t->entries.size());
    if (grow > 0) {
      need += grow;
    } else {
      const uint32_t page = t->entries[pos / ps];
      if (page >= pool->capacity) return pkv::fail(PKV_INDEX_ERROR, "page out of bounds");
      if (pool->ref(page) > 1) need += 1;  // copy-on-write
    }
  }
  const int64_t avail = static_cast<int64_t>(pool->free_stack.size()) +
                        static_cast<int64_t>(pool->capacity - pool->bump_cursor());
  if (need > avail)
    return pkv::fail(PKV_CAPACITY_EXHAUSTED, "decode step needs %lld pages, %lld available",
                     static_cast<long long>(need), static_cast<long long>(avail));
  if (need > pages_cap) return pkv::fail(PKV_VALUE_ERROR, "pages_out too small");
  // phase 2: apply (cannot fail)
  pkv_append_undo* undo = nullptr;
  if (undo_out) {
    undo = new pkv_append_undo;
    undo->stack_size = pool->free_stack.size();
    const size_t k = std::min<size_t>(static_cast<size_t>(need), undo->stack_size);
    undo->stack_tail.assign(pool->free_stack.end() - k, pool->free_stack.end());
    undo->bump_raw = pool->bump_raw;
    undo->seqs.reserve(n);
  }
  int64_t np = 0;
  std::vector<uint32_t> got;
  for (int64_t i = 0; i < n; ++i) {
    Table& t = *tabs[i];
    const int64_t pos = t.logical_len;
    if (undo) undo->seqs.push_back({seqs[i], pos, t.entries.size(), -1, 0});
    copies_out[2 * i] = copies_out[2 * i + 1] = -1;
    const int64_t grow = pool->pages_for(pos + 1) - static_cast<int64_t>(t.entries.size());
    if (grow > 0) {
      pool->take(grow, &got);
      for (uint32_t p : got) {
        pool->set_ref(p, 1);
        pages_out[np++] = p;
      }
      pool->append_entries(t, got);
    } else {
      const int64_t blk = pos / ps;
      const uint32_t old = t.entries[blk];
      if (pool->ref(old) > 1) {
        pool->take(1, &got);
        pool->set_ref(got[0], 1);
        t.entries[blk] = got[0];
        pool->mark(t, blk);
        int64_t dummy;
        pool->release(std::vector<uint32_t>{old}, &dummy);
        copies_out[2 * i] = old;
        copies_out[2 * i + 1] = got[0];
        if (undo) {
          undo->seqs.back().cow_block = blk;
          undo->seqs.back().cow_old = old;
          undo->granted.push_back(got[0]);
        }
      }
    }
    positions_out[i] = static_cast<int32_t>(pos);
    rows_out[i] = t.mirror_row;
    t.logical_len = pos + 1;
  }
  if (undo) undo->granted.insert(undo->granted.end(), pages_out, pages_out + np);
  *n_pages_out = np;
  if (undo_out) *undo_out = undo;
  return PKV_OK;
}

int pkv_pool_rollback_append(pkv_pool* pool, pkv_append_undo* undo) {
  if (!undo) return PKV_OK;
  std::unique_ptr<pkv_append_undo> hold(undo);
  LOCK_MUT(pool);
  for (auto it = undo->seqs.rbegin(); it != undo->seqs.rend(); ++it) {
    Table* t = pool->find(it->handle);
    if (!t) return pkv::fail(PKV_UNKNOWN_SEQUENCE, "rollback: table %lld vanished", static_cast<long long>(it->handle));
    if (it->cow_block >= 0) {
      pool->set_ref(it->cow_old, pool->ref(it->cow_old) + 1);
      t->entries[it->cow_block] = it->cow_old;
      pool->mark(*t, it->cow_block);
    }
    for (size_t c = it->n_entries; c < t->entries.size(); ++c) {  // clear the grown columns
      const int64_t flat = t->mirror_row * pool->mcols + static_cast<int64_t>(c);
      pool->mirror[flat] = 0;
      if (!pool->full_resync) pool->dirty.push_back(flat);
    }
    t->entries.resize(it->n_entries);
    t->logical_len = it->logical_len;
  }
  for (uint32_t p : undo->granted) pool->set_ref(p, 0);
  pool->free_stack.resize(undo->stack_size - undo->stack_tail.size());
  pool->free_stack.insert(pool->free_stack.end(), undo->stack_tail.begin(), undo->stack_tail.end());
  pool->bump_raw = undo->bump_raw;
  return PKV_OK;
}

void pkv_pool_release_undo(pkv_append_undo* undo) { delete undo; }

extern "C" {

int pkv_pool_translate(pkv_pool* pool, int64_t seq, int64_t position, uint32_t* page_out,
                       uint32_t* offset_out) {
  LOCK(pool);
  TABLE_OR_FAIL(t, pool, seq);
  const int64_t ps = pool->page_size;
  int64_t blk = floordiv(position, ps);
  if (position < 0 || blk >= static_cast<int64_t>(t->entries.size()))
    return pkv::fail(PKV_OUT_OF_RANGE, "position %lld outside reserved capacity %lld",
                     static_cast<long long>(position),
                     static_cast<long long>(t->entries.size() * ps));
  if (page_out) *page_out = t->entries[blk];
  if (offset_out) *offset_out = static_cast<uint32_t>(position - blk * ps);
  return PKV_OK;
}

int pkv_pool_has_sequence(pkv_pool* pool, int64_t seq, int32_t* out) {
  LOCK(pool);
  *out = pool->find(seq) != nullptr;
  return PKV_OK;
}

int pkv_pool_table_len(pkv_pool* pool, int64_t seq, int64_t* n_out) {
  LOCK(pool);
  TABLE_OR_FAIL(t, pool, seq);
  *n_out = static_cast<int64_t>(t->entries.size());
  return PKV_OK;
}

int pkv_pool_table_entries(pkv_pool* pool, int64_t seq, uint32_t* out, int64_t cap) {
  LOCK(pool);
  TABLE_OR_FAIL(t, pool, seq);
  if (cap < static_cast<int64_t>(t->entries.size()))
    return pkv::fail(PKV_VALUE_ERROR, "output buffer too small");
  copy_out(t->entries, out, nullptr);
  return PKV_OK;
}

int pkv_pool_table_set_entry(pkv_pool* pool, int64_t seq, int64_t idx, uint32_t value) {
  LOCK_MUT(pool);
  TABLE_OR_FAIL(t, pool, seq);
  const int64_t n = static_cast<int64_t>(t->entries.size());
  if (idx < 0) idx += n;
  if (idx < 0 || idx >= n) return pkv::fail(PKV_INDEX_ERROR, "array assignment index out of range");
  t->entries[idx] = value;
  pool->mark(*t, idx);
  return PKV_OK;
}

int pkv_pool_get_logical_len(pkv_pool* pool, int64_t seq, int64_t* out) {
  LOCK(pool);
  TABLE_OR_FAIL(t, pool, seq);
  *out = t->logical_len;
  return PKV_OK;
}

int pkv_pool_set_logical_len(pkv_pool* pool, int64_t seq, int64_t value) {
  LOCK_MUT(pool);
  TABLE_OR_FAIL(t, pool, seq);
  t->logical_len = value;
  return PKV_OK;
}

int pkv_pool_sequence_count(pkv_pool* pool, int64_t* n_out) {
  LOCK(pool);
  *n_out = static_cast<int64_t>(pool->tables.size());
  return PKV_OK;
}

int pkv_pool_sequences(pkv_pool* pool, int64_t* out, int64_t cap) {
  LOCK(pool);
  if (cap < static_cast<int64_t>(pool->tables.size()))
    return pkv::fail(PKV_VALUE_ERROR, "output buffer too small");
  std::vector<std::pair<uint64_t, int64_t>> v;
  v.reserve(pool->tables.size());
  for (auto& kv : pool->tables) v.emplace_back(kv.second.order, kv.first);
  std::sort(v.begin(), v.end());
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i].second;
  return PKV_OK;
}

int pkv_pool_refcount(pkv_pool* pool, uint64_t page, int64_t* out) {
  LOCK(pool);
  if (page >= pool->capacity) return pkv::fail(PKV_INDEX_ERROR, "page out of bounds");
  *out = pool->ref(page);
  return PKV_OK;
}

int pkv_pool_census(pkv_pool* pool, int64_t* out5) {
  LOCK(pool);
  out5[0] = static_cast<int64_t>(pool->capacity);
  out5[1] = pool->nonzero;
  out5[2] = static_cast<int64_t>(pool->free_stack.size());
  out5[3] = static_cast<int64_t>(pool->capacity - pool->bump_cursor());
  out5[4] = static_cast<int64_t>(pool->bump_cursor());
  return PKV_OK;
}

int pkv_pool_free_stack(pkv_pool* pool, uint32_t* out, int64_t cap, int64_t* n_out) {
  LOCK(pool);
  *n_out = static_cast<int64_t>(pool->free_stack.size());
  if (out) {
    if (cap < *n_out) return pkv::fail(PKV_VALUE_ERROR, "output buffer too small");
    copy_out(pool->free_stack, out, nullptr);
  }
  return PKV_OK;
}

int pkv_pool_generation(pkv_pool* pool, uint64_t* out) {
  if (!pool) return pkv::fail(PKV_VALUE_ERROR, "null pool handle");
  *out = pool->generation.load(std::memory_order_relaxed);
  return PKV_OK;
}

int pkv_pool_mirror_row(pkv_pool* pool, int64_t seq, int32_t* row_out) {
  LOCK(pool);
  TABLE_OR_FAIL(t, pool, seq);
  *row_out = t->mirror_row;
  return PKV_OK;
}

int pkv_pool_tables_info(pkv_pool* pool, const int64_t* seqs, int64_t n, int64_t* n_pages_out,
                         int32_t* mirror_row_out) {
  if (n < 0 || (n > 0 && !seqs)) return pkv::fail(PKV_VALUE_ERROR, "bad sequence list");
  LOCK(pool);
  for (int64_t i = 0; i < n; ++i) {
    TABLE_OR_FAIL(t, pool, seqs[i]);
    if (n_pages_out) n_pages_out[i] = static_cast<int64_t>(t->entries.size());
    if (mirror_row_out) mirror_row_out[i] = t->mirror_row;
  }
  return PKV_OK;
}

int pkv_pool_mirror_shape(pkv_pool* pool, int64_t* rows_out, int64_t* cols_out) {
  LOCK(pool);
  pool->ensure_shape(1, 1);
  *rows_out = pool->mrows;
  *cols_out = pool->mcols;
  return PKV_OK;
}

int pkv_pool_mirror_pending(pkv_pool* pool, int64_t* n_out, int32_t* full_resync) {
  LOCK(pool);
  *n_out = static_cast<int64_t>(pool->dirty.size());
  *full_resync = pool->full_resync;
  return PKV_OK;
}

int pkv_pool_mirror_drain(pkv_pool* pool, int32_t* pairs_out, int64_t cap, int64_t* n_out,
                          int32_t* full_resync) {
  LOCK(pool);
  *n_out = 0;
  *full_resync = pool->full_resync;
  if (pool->full_resync) return PKV_OK;  // caller must export the whole matrix
  int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(pool->dirty.size()));
  for (int64_t i = 0; i < n; ++i) {
    int64_t flat = pool->dirty[i];
    pairs_out[2 * i] = static_cast<int32_t>(flat);
    pairs_out[2 * i + 1] = pool->mirror[flat];
  }
  pool->dirty.erase(pool->dirty.begin(), pool->dirty.begin() + n);
  *n_out = n;
  return PKV_OK;
}

int pkv_pool_mirror_export(pkv_pool* pool, int32_t* out, int64_t rows, int64_t cols) {
  LOCK(pool);
  pool->ensure_shape(1, 1);
  if (rows != pool->mrows || cols != pool->mcols)
    return pkv::fail(PKV_SHAPE_MISMATCH, "mirror is %lld x %lld, caller passed %lld x %lld",
                     static_cast<long long>(pool->mrows), static_cast<long long>(pool->mcols),
                     static_cast<long long>(rows), static_cast<long long>(cols));
  std::memcpy(out, pool->mirror.data(), sizeof(int32_t) * rows * cols);
  pool->dirty.clear();
  pool->full_resync = false;
  return PKV_OK;
}

}  // extern "C"
