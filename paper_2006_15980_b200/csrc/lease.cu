// Node-local column-lease table for the multi-GPU engine (host code).
//
// The reference grants leases under one in-process Condition
// (scheduler.py:333-409): a worker takes a unit whose row and column are
// free, and releases it when its update is done.  Across the processes of
// one B200 node (one per GPU) the column leases of distributed.RowBandTrainer
// live here instead of on the torch.distributed TCPStore: a POSIX
// shared-memory segment holding, per column band, the holder (-1 = free) and
// the last owner (whose Q replica holds the band's newest rows), plus a
// global ticket counter.  Every operation is one lock-free atomic on a
// cache line of its own — ~0.1 us against ~50-100 us per TCPStore round
// trip (three to four of them per lease).
//
// Ordering: release() publishes the new owner before freeing the lease
// (release store, then a CAS with release semantics); try_acquire's CAS has
// acquire semantics, so whoever wins the lease next reads the owner that
// released it.
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "hmf_internal.h"

namespace hmf {
namespace lease {

constexpr uint64_t kMagic = 0x484D464C45415345ULL;  // "HMFLEASE"

struct alignas(64) Slot {
  std::atomic<int32_t> holder;  // rank holding the lease, -1 = free
  std::atomic<int32_t> owner;   // rank whose replica holds the newest rows, -1 = any
};

struct alignas(64) Header {
  std::atomic<uint64_t> magic;
  int32_t n_cols;
  int32_t pad;
  alignas(64) std::atomic<int64_t> seq;
  alignas(64) std::atomic<int64_t> ops;  // atomic operations served (all ranks)
  // 0, or 1 + the rank that aborted the run (scheduler.abort,
  // scheduler.py:415-423 / workers.py:300-302): acquires fail from then on
  alignas(64) std::atomic<int32_t> aborted;
  // block updates claimed so far (the free policy's job-wide epoch counter)
  alignas(64) std::atomic<int64_t> work;
};

static_assert(std::atomic<int32_t>::is_always_lock_free, "address-free atomics needed");
static_assert(std::atomic<int64_t>::is_always_lock_free, "address-free atomics needed");

struct Table {
  Header* h;
  Slot* slots;
  size_t bytes;
  char name[128];
};

static size_t segment_bytes(int32_t n_cols) {
  return sizeof(Header) + size_t(n_cols) * sizeof(Slot);
}

static Table* checked(void* t, int32_t c) {
  Table* tb = static_cast<Table*>(t);
  if (!tb) {
    set_error(HMF_ERR_ARG, "null lease table");
    return nullptr;
  }
  if (c < 0 || c >= tb->h->n_cols) {
    set_error(HMF_ERR_ARG, "column out of range");
    return nullptr;
  }
  return tb;
}

// HMF_ERR_ABORTED with the aborting rank in the message once the run is aborted
static bool aborted_error(Table* t) {
  const int32_t a = t->h->aborted.load(std::memory_order_acquire);
  if (!a) return false;
  char msg[96];
  std::snprintf(msg, sizeof(msg), "the run was aborted by rank %d", a - 1);
  set_error(HMF_ERR_ABORTED, msg);
  return true;
}

}  // namespace lease
}  // namespace hmf

extern "C" {

int hmf_lease_open(const char* name, int32_t n_cols, int32_t create, void** out) {
  using namespace hmf::lease;
  if (!name || !out || name[0] != '/' || std::strlen(name) >= sizeof(Table::name))
    return int(hmf::set_error(HMF_ERR_ARG, "lease table name must be '/...' (< 128 chars)"));
  if (n_cols <= 0) return int(hmf::set_error(HMF_ERR_ARG, "n_cols must be > 0"));
  *out = nullptr;
  const size_t bytes = segment_bytes(n_cols);
  int fd;
  if (create) {
    shm_unlink(name);  // a stale segment of an earlier run with this name
    fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd >= 0 && ftruncate(fd, off_t(bytes)) != 0) {
      close(fd);
      shm_unlink(name);
      fd = -1;
    }
  } else {
    fd = shm_open(name, O_RDWR, 0600);
  }
  if (fd < 0) {
    char msg[200];
    std::snprintf(msg, sizeof(msg), "shm_open(%s): %s", name, std::strerror(errno));
    return int(hmf::set_error(HMF_ERR_ARG, msg));
  }
  struct stat st;
  if (fstat(fd, &st) != 0 || size_t(st.st_size) < bytes) {
    close(fd);
    return int(hmf::set_error(HMF_ERR_ARG, "lease table segment too small (not initialised?)"));
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return int(hmf::set_error(HMF_ERR_ARG, "mmap of the lease table failed"));
  Table* t = new Table;
  t->h = static_cast<Header*>(p);
  t->slots = reinterpret_cast<Slot*>(static_cast<unsigned char*>(p) + sizeof(Header));
  t->bytes = bytes;
  std::snprintf(t->name, sizeof(t->name), "%s", name);
  if (create) {
    t->h->n_cols = n_cols;
    t->h->seq.store(0, std::memory_order_relaxed);
    t->h->ops.store(0, std::memory_order_relaxed);
    t->h->aborted.store(0, std::memory_order_relaxed);
    t->h->work.store(0, std::memory_order_relaxed);
    for (int32_t c = 0; c < n_cols; ++c) {
      t->slots[c].holder.store(-1, std::memory_order_relaxed);
      t->slots[c].owner.store(-1, std::memory_order_relaxed);
    }
    t->h->magic.store(kMagic, std::memory_order_release);
  } else if (t->h->magic.load(std::memory_order_acquire) != kMagic || t->h->n_cols != n_cols) {
    munmap(p, bytes);
    delete t;
    return int(hmf::set_error(HMF_ERR_ARG, "lease table segment: bad magic or column count"));
  }
  *out = t;
  return HMF_OK;
}

int hmf_lease_close(void* table, int32_t unlink_segment) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return HMF_OK;
  if (unlink_segment) shm_unlink(t->name);
  munmap(t->h, t->bytes);
  delete t;
  return HMF_OK;
}

int32_t hmf_lease_try_acquire(void* table, int32_t c, int32_t rank) {
  using namespace hmf::lease;
  Table* t = checked(table, c);
  if (!t) return HMF_ERR_ARG;
  if (rank < 0) return int32_t(hmf::set_error(HMF_ERR_ARG, "rank must be >= 0"));
  if (aborted_error(t)) return HMF_ERR_ABORTED;
  t->h->ops.fetch_add(1, std::memory_order_relaxed);
  int32_t expect = -1;
  return t->slots[c].holder.compare_exchange_strong(expect, rank, std::memory_order_acq_rel,
                                                    std::memory_order_acquire)
             ? 1
             : 0;
}

int hmf_lease_acquire_first(void* table, const int32_t* cands, int32_t n, int32_t rank,
                            int32_t* got) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t || !got || (!cands && n > 0)) return int(hmf::set_error(HMF_ERR_ARG, "null argument"));
  if (rank < 0) return int(hmf::set_error(HMF_ERR_ARG, "rank must be >= 0"));
  *got = -1;
  if (aborted_error(t)) return HMF_ERR_ABORTED;
  for (int32_t i = 0; i < n; ++i)
    if (cands[i] < 0 || cands[i] >= t->h->n_cols)
      return int(hmf::set_error(HMF_ERR_ARG, "column out of range"));
  for (int32_t i = 0; i < n; ++i) {
    const int32_t c = cands[i];
    // a plain load first: a busy column costs no cache-line ownership transfer
    if (t->slots[c].holder.load(std::memory_order_relaxed) != -1) continue;
    t->h->ops.fetch_add(1, std::memory_order_relaxed);
    int32_t expect = -1;
    if (t->slots[c].holder.compare_exchange_strong(expect, rank, std::memory_order_acq_rel,
                                                   std::memory_order_acquire)) {
      *got = c;
      return HMF_OK;
    }
  }
  return HMF_OK;
}

int32_t hmf_lease_release(void* table, int32_t c, int32_t rank) {
  using namespace hmf::lease;
  Table* t = checked(table, c);
  if (!t) return HMF_ERR_ARG;
  t->h->ops.fetch_add(1, std::memory_order_relaxed);
  // only the holder frees a lease, so this check cannot go stale before the
  // CAS; it keeps a bad release from touching the owner
  if (t->slots[c].holder.load(std::memory_order_acquire) != rank) {
    char msg[96];
    std::snprintf(msg, sizeof(msg), "rank %d released column %d it did not hold", rank, c);
    return int32_t(hmf::set_error(HMF_ERR_ARG, msg));
  }
  // publish the new owner first: whoever leases c next pulls from us
  t->slots[c].owner.store(rank, std::memory_order_release);
  int32_t expect = rank;
  t->slots[c].holder.compare_exchange_strong(expect, -1, std::memory_order_acq_rel,
                                             std::memory_order_acquire);
  return HMF_OK;
}

int hmf_lease_owner(void* table, int32_t c, int32_t* owner) {
  using namespace hmf::lease;
  Table* t = checked(table, c);
  if (!t) return HMF_ERR_ARG;
  if (!owner) return int(hmf::set_error(HMF_ERR_ARG, "null argument"));
  *owner = t->slots[c].owner.load(std::memory_order_acquire);
  return HMF_OK;
}

int hmf_lease_holder(void* table, int32_t c, int32_t* holder) {
  using namespace hmf::lease;
  Table* t = checked(table, c);
  if (!t) return HMF_ERR_ARG;
  if (!holder) return int(hmf::set_error(HMF_ERR_ARG, "null argument"));
  *holder = t->slots[c].holder.load(std::memory_order_acquire);
  return HMF_OK;
}

int64_t hmf_lease_ticket(void* table) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return hmf::set_error(HMF_ERR_ARG, "null lease table");
  t->h->ops.fetch_add(1, std::memory_order_relaxed);
  return t->h->seq.fetch_add(1, std::memory_order_acq_rel) + 1;
}

int64_t hmf_lease_claim(void* table, int64_t target) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return hmf::set_error(HMF_ERR_ARG, "null lease table");
  if (aborted_error(t)) return HMF_ERR_ABORTED;
  t->h->ops.fetch_add(1, std::memory_order_relaxed);
  int64_t old = t->h->work.load(std::memory_order_acquire);
  while (old < target) {
    if (t->h->work.compare_exchange_weak(old, old + 1, std::memory_order_acq_rel,
                                         std::memory_order_acquire))
      return old + 1;
  }
  return 0;
}

int hmf_lease_abort(void* table, int32_t rank) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return int(hmf::set_error(HMF_ERR_ARG, "null lease table"));
  int32_t expect = 0;
  t->h->aborted.compare_exchange_strong(expect, rank + 1, std::memory_order_acq_rel);
  return HMF_OK;
}

int32_t hmf_lease_aborted(void* table) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return int32_t(hmf::set_error(HMF_ERR_ARG, "null lease table"));
  return t->h->aborted.load(std::memory_order_acquire) - 1;
}

int64_t hmf_lease_ops(void* table) {
  using namespace hmf::lease;
  Table* t = static_cast<Table*>(table);
  if (!t) return hmf::set_error(HMF_ERR_ARG, "null lease table");
  return t->h->ops.load(std::memory_order_relaxed);
}

}  // extern "C"
