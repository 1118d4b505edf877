// driver.cu — host driver and C ABI of libsexpm (see include/sexpm.h).
//
// Algorithm 4.2 on one or more B200s.  Host work is scalar only
// (Eq. 4.20 enumeration, Algorithm 4.1's threshold recurrence); every matrix step runs
// in the kernels of kernels.cu.  Multi-GPU: contiguous row blocks, NCCL halo exchange of
// the rows of T^_{i-1} within its bandwidth (Lemma 3.1) and tiny scalar
// all-gathers summed in rank order (identical thresholds on every rank).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <memory>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sexpm.h"
#include "kernels.cuh"

using namespace sx;

// ------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------
static thread_local std::string g_err;

struct SxError {
  int code;
  std::string msg;
};

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw SxError{e_ == cudaErrorMemoryAllocation ? SEXPM_ENOMEM : SEXPM_ECUDA,       \
                    std::string(#x) + ": " + cudaGetErrorString(e_)};                   \
  } while (0)

#define REQUIRE(cond, code, msg)                \
  do {                                          \
    if (!(cond)) throw SxError{(code), (msg)};  \
  } while (0)

// ------------------------------------------------------------------------------------
// NCCL, loaded at run time (the library works on one GPU without NCCL present)
// ------------------------------------------------------------------------------------
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Bcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                        cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*ErrStr)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;

static NcclApi &nccl() {
  if (!g_nccl.tried) {
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define NS(f, s) g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, s))
      NS(GetUniqueId, "ncclGetUniqueId");
      NS(CommInitRank, "ncclCommInitRank");
      NS(CommDestroy, "ncclCommDestroy");
      NS(AllGather, "ncclAllGather");
      NS(Send, "ncclSend");
      NS(Recv, "ncclRecv");
      NS(Bcast, "ncclBroadcast");
      NS(GroupStart, "ncclGroupStart");
      NS(GroupEnd, "ncclGroupEnd");
      NS(ErrStr, "ncclGetErrorString");
#undef NS
      g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather &&
                  g_nccl.Send && g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd &&
                  g_nccl.Bcast;
    }
  }
  REQUIRE(g_nccl.ok, SEXPM_ENCCL, "libnccl.so.2 could not be loaded");
  return g_nccl;
}

#define NK(x)                                                                            \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      throw SxError{SEXPM_ENCCL, std::string(#x) + ": " +                                \
                                     (g_nccl.ErrStr ? g_nccl.ErrStr(r_) : "nccl error")}; \
  } while (0)

// ------------------------------------------------------------------------------------
// Transport between the ranks of a row-partitioned plan: an all-gather
// of equal-size pieces and a group of point-to-point transfers.  NcclTransport runs them over
// NCCL (one process per GPU, NVLink / NVSwitch); VirtualTransport runs W ranks as host threads
// of one process on one device (the multi-rank code path executed and tested on a single
// GPU): every call is a host barrier, then device-to-device copies out of the peers' posted
// buffers on the caller's stream, then a second barrier.  No kernel ever waits on another
// rank: the waiting is on the host.
// ------------------------------------------------------------------------------------
struct Transport {
  int world = 1, rank = 0;
  struct Xfer {
    int peer;
    const void *src;
    void *dst;
    size_t bytes;
  };
  virtual ~Transport() = default;
  // recv[g * bytes .. (g+1) * bytes) = rank g's send (device pointers, all ranks the same size)
  virtual void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;
  // sends[k] goes to sends[k].peer, recvs[k] comes from recvs[k].peer; the transfers between a
  // pair of ranks are matched in the order listed (src / dst of sends / recvs respectively)
  virtual void exchange(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs,
                        cudaStream_t st) = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    NK(nccl().AllGather(send, recv, bytes, ncclChar, comm, st));
  }
  void exchange(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs,
                cudaStream_t st) override {
    NK(nccl().GroupStart());
    for (const Xfer &x : sends)
      if (x.bytes) NK(nccl().Send(x.src, x.bytes, ncclChar, x.peer, comm, st));
    for (const Xfer &x : recvs)
      if (x.bytes) NK(nccl().Recv(x.dst, x.bytes, ncclChar, x.peer, comm, st));
    NK(nccl().GroupEnd());
  }
};

struct VirtualHub {
  int W = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void *> ag;                   // posted all-gather sources
  std::vector<std::vector<Transport::Xfer>> sent;  // posted sends per rank
  std::atomic<int> refs{0};
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == W) {
      arrived = 0;
      gen++;
      cv.notify_all();
      return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; });
    REQUIRE(ok, SEXPM_ENCCL, "virtual transport: a rank did not arrive within 300 s");
  }
};

struct VirtualTransport : Transport {
  VirtualHub *hub = nullptr;
  void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));  // the piece is complete before peers read it
    hub->ag[rank] = send;
    hub->barrier();
    for (int g = 0; g < world; g++)
      if (bytes) CK(cudaMemcpyAsync((char *)recv + (size_t)g * bytes, hub->ag[g], bytes, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    hub->barrier();  // nobody reuses its send buffer before every peer has read it
  }
  void exchange(const std::vector<Xfer> &sends, const std::vector<Xfer> &recvs,
                cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    hub->sent[rank] = sends;
    hub->barrier();
    std::vector<size_t> next((size_t)world, 0);  // next unmatched send of each peer to me
    for (const Xfer &r : recvs) {
      const std::vector<Xfer> &ps = hub->sent[r.peer];
      size_t &k = next[r.peer];
      while (k < ps.size() && ps[k].peer != rank) k++;
      REQUIRE(k < ps.size() && ps[k].bytes == r.bytes, SEXPM_EINTERNAL,
              "virtual transport: receive without a matching send");
      if (r.bytes) CK(cudaMemcpyAsync(r.dst, ps[k].src, r.bytes, cudaMemcpyDeviceToDevice, st));
      k++;
    }
    CK(cudaStreamSynchronize(st));
    hub->barrier();
  }
};

// the communicator handle of the C ABI (sexpm_nccl_comm_init / sexpm_virtual_comm_create)
struct SxComm {
  uint64_t magic = 0x53584d434f4d4d31ull;  // "SXMCOMM1"
  int kind = 0;                           // 0 NCCL, 1 virtual
  int world = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  VirtualHub *hub = nullptr;
};
static SxComm *as_comm(void *h) {
  SxComm *c = reinterpret_cast<SxComm *>(h);
  REQUIRE(c && c->magic == 0x53584d434f4d4d31ull, SEXPM_EINVAL,
          "options.nccl_comm is not a handle from sexpm_nccl_comm_init / sexpm_virtual_comm_create");
  return c;
}

// ------------------------------------------------------------------------------------
// device buffers (stream-ordered allocator)
// ------------------------------------------------------------------------------------
// Process-wide cache of device blocks.  Every plan grows its iterates and staging pool
// as the terms fill in, and a new plan starts empty; mapping fresh memory through the
// stream-ordered pool costs ~20-30 ms per GB, so freed blocks are kept here and handed
// to later requests (best fit within 2x).  A block freed while its stream still has work
// queued is reused only on that stream (stream order makes that safe); blocks freed after
// a synchronize (sexpm_destroy) are idle and reusable on any stream.
namespace cache {
struct Block {
  void *p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;  // nullptr: idle (no pending work)
  int dev = 0;
};
static std::mutex mu;
static std::multimap<size_t, Block> free_blocks;
static long long hits = 0, misses = 0, releases = 0;
static double bytes_cached = 0.0, bytes_allocated = 0.0;
static size_t budget = 0;  // cap on bytes_allocated: 90% of the device memory
static thread_local bool freeing_idle = false;
// Role parking: the final block of each role-tagged buffer (iterates, staging pool, E) of a
// destroyed plan is kept for the same role of the next plan, which takes it whenever it is
// large enough for its first request: a plan on a matrix like the previous one gets its
// final-size buffers at once, with no cross-role fragmentation.
constexpr int kRoles = 64;
static Block parked[kRoles];
static size_t round_bytes(size_t b) {
  const size_t g = b >= ((size_t)1 << 24) ? ((size_t)1 << 21) : 512;
  return (b + g - 1) / g * g;
}
static void free_block(const Block &b, cudaStream_t fallback) {  // mu held
  cudaFreeAsync(b.p, b.st ? b.st : fallback);
  bytes_allocated -= (double)b.bytes;
  bytes_cached -= (double)b.bytes;
}
static void release_all() {
  std::lock_guard<std::mutex> lk(mu);
  for (auto &kv : free_blocks) {
    if (kv.second.st) cudaFreeAsync(kv.second.p, kv.second.st);
    else cudaFree(kv.second.p);
    bytes_allocated -= (double)kv.first;
  }
  free_blocks.clear();
  for (Block &b : parked) {
    if (b.p) {
      cudaFree(b.p);
      bytes_allocated -= (double)b.bytes;
    }
    b = Block{};
  }
  bytes_cached = 0.0;
  releases++;
}
// blocks whose stream has just been synchronized carry no pending work
static void mark_idle(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(mu);
  for (auto &kv : free_blocks)
    if (kv.second.st == st) kv.second.st = nullptr;
}
static bool take(size_t lo, size_t hi, cudaStream_t st, int dev, void **p, size_t *got) {
  for (auto it = free_blocks.lower_bound(lo); it != free_blocks.end() && it->first <= hi; ++it) {
    if (it->second.dev == dev && (it->second.st == st || it->second.st == nullptr)) {
      *p = it->second.p;
      *got = it->first;
      bytes_cached -= (double)it->first;
      free_blocks.erase(it);
      hits++;
      return true;
    }
  }
  return false;
}
static void *alloc(size_t bytes, cudaStream_t st, size_t *got) {
  bytes = round_bytes(bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  void *p = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (budget == 0) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      budget = (size_t)(0.90 * (double)tot);
    }
    if (take(bytes, 2 * bytes + ((size_t)1 << 21), st, dev, &p, got)) return p;
    // miss: make room under the budget by returning the largest cached blocks to the pool
    while (!free_blocks.empty() && bytes_allocated + (double)bytes > (double)budget) {
      auto it = std::prev(free_blocks.end());
      free_block(it->second, st);
      free_blocks.erase(it);
    }
  }
  cudaError_t e = cudaMallocAsync(&p, bytes, st);
  if (e == cudaErrorMemoryAllocation) {  // give everything cached back, trim the pool, retry
    cudaGetLastError();
    cudaStreamSynchronize(st);
    release_all();
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&p, bytes, st);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw SxError{e == cudaErrorMemoryAllocation ? SEXPM_ENOMEM : SEXPM_ECUDA,
                  std::string("device allocation of ") + std::to_string(bytes) + " bytes: " +
                      cudaGetErrorString(e)};
  }
  *got = bytes;
  {
    std::lock_guard<std::mutex> lk(mu);
    misses++;
    bytes_allocated += (double)bytes;
  }
  if (getenv("SEXPM_CACHE_LOG"))
    fprintf(stderr, "[sexpm cache] miss: %zu bytes, allocated %.1f GB, cached %.1f GB\n", bytes,
            bytes_allocated / 1e9, bytes_cached / 1e9);
  return p;
}
// very large blocks that are not parked (growth trails of a cold plan) go back to the CUDA
// pool at once: only the parked final blocks and blocks under 1 GiB are kept (config 5 takes
// eight 80-370 MB work buffers per plan: re-allocating them every plan cost 8 misses and an
// occasional 100+ ms stall in cudaMallocAsync at 136 GB allocated)
constexpr size_t kKeepMax = (size_t)1 << 30;
static void free(void *p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (bytes >= kKeepMax) {
    if (freeing_idle || st == nullptr) cudaFree(p);
    else cudaFreeAsync(p, st);
    bytes_allocated -= (double)bytes;
    return;
  }
  free_blocks.emplace(bytes, Block{p, bytes, freeing_idle ? nullptr : st, dev});
  bytes_cached += (double)bytes;
}
static void park(int role, void *p, size_t bytes) {  // idle blocks only (plan destroyed)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Block &b = parked[role];
  Block other{p, bytes, nullptr, dev};
  if (!b.p || (b.bytes < bytes && b.dev == dev)) std::swap(b, other);  // keep the larger one
  if (other.p) {  // the smaller block of a role goes back to the pool
    cudaFree(other.p);
    bytes_allocated -= (double)other.bytes;
  }
}
// bytes parked for a role (reused by its next ensure when large enough); caller holds mu
static size_t parked_bytes(int role) {
  int dev = 0;
  cudaGetDevice(&dev);
  return (role >= 0 && parked[role].p && parked[role].dev == dev) ? parked[role].bytes : 0;
}
static void *unpark(int role, size_t bytes, size_t *got) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Block &b = parked[role];
  if (b.p && b.dev == dev && b.bytes >= round_bytes(bytes)) {
    void *p = b.p;
    *got = b.bytes;
    b = Block{};
    hits++;
    return p;
  }
  return nullptr;
}
}  // namespace cache

template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  int role = -1;      // cache::parked slot (large growing buffers), -1 none
  bool grown = false;  // allocated at least once in this plan
  void release() {
    if (p) {
      if (role >= 0 && cache::freeing_idle) cache::park(role, p, bytes);  // plan destroyed
      else cache::free(p, bytes, st);
    }
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  void alloc(size_t cnt, cudaStream_t s) {
    release();
    st = s;
    if (cnt == 0) cnt = 1;
    p = nullptr;
    if (role >= 0 && !grown) p = reinterpret_cast<T *>(cache::unpark(role, cnt * sizeof(T), &bytes));
    if (!p) p = reinterpret_cast<T *>(cache::alloc(cnt * sizeof(T), s, &bytes));
    n = bytes / sizeof(T);
    grown = true;
  }
  // grow-only: reuse the buffer when it is large enough, else grow by 1.25x; the large
  // role-tagged buffers (iterates, staging pool), which fill in term after term, at least
  // double, so a cold plan re-allocates them a few times rather than at every step
  void ensure(size_t cnt, cudaStream_t s) {
    if (cnt > n || !p) alloc(std::max<size_t>(cnt + cnt / 4, 1), s);
  }
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept { *this = std::move(o); }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      bytes = o.bytes;
      st = o.st;
      grown = o.grown;  // role stays with the slot (swap_csr keeps roles per slot)
      o.p = nullptr;
      o.n = 0;
      o.bytes = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
};

struct DCsr {
  int64_t nrows = 0, row0 = 0, nnz = 0;
  DBuf<int64_t> rp;
  DBuf<int32_t> col;
  DBuf<double> val;
  // padded form (the Taylor accumulator T^_0): row r holds len[r] entries from rp[r], rp[r+1]
  // is a capacity bound; nnz is the capacity
  bool padded = false;
  DBuf<int64_t> len;
  CsrView view() const {
    CsrView v;
    v.nrows = nrows;
    v.row0 = row0;
    v.nnz = nnz;
    v.rp = rp.p;
    v.col = col.p;
    v.val = val.p;
    return v;
  }
};

static CsrView view_of(const sexpm_csr_in *H, int64_t row0_override = -1) {
  CsrView v;
  v.nrows = H->row_end - H->row_begin;
  v.row0 = row0_override >= 0 ? row0_override : H->row_begin;
  v.nnz = H->nnz;
  v.rp = H->rowptr;
  v.col = H->colidx;
  v.val = H->vals;
  return v;
}

// ------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------
struct StepReport {
  int32_t passes = 0;
  double tau = 0.0, fsum = 0.0;
  int64_t nnz_unf = 0, staged = 0, nnz = 0;
  double normIT2 = 0.0;
  int64_t l1 = 0, l2 = 0;
  double fmas = 0.0;
  float numeric_ms = 0.f;
  double numeric_bytes = 0.0;
  int64_t window_rows = 0;
  float first_ms = 0.f;  // the first kernel of the fallback chain alone
  float kernel_ms = 0.f;  // the block kernel alone (kernel 11), else 0
  int64_t bsr_blocks = 0;  // blocks of the BSR-8 view (kernel 11)
  double block_products = 0.0;  // 8x8 block products executed (kernel 11)
  unsigned long long prof[12] = {0};  // grouped kernel phase clocks
  float asm_ms = 0.f;  // symmetric path: K3c + K3a
  bool sym = false;    // the product ran on the symmetric path
  bool relabel_needed = false;  // T^_0 in index order could not take the symmetric path
  bool need_csr = false;        // T^ in block form could not take the symmetric path
};

// BSR-8 view of a CSR matrix (k_bsr_build) and, optionally, its block transpose
struct BsrBufs {
  DBuf<int64_t> bcnt, brp, tp, cnt64, tb, tb_tmp;
  DBuf<int32_t> bcol, tcnt, tk, tk_tmp, keys_tmp;
  DBuf<double> bval;
  DBuf<unsigned char> sort_tmp;
  int64_t nbr = 0, nb = 0, bmax = 0;
  bool frag = false, transposed = false;
  BsrView view() const {
    BsrView v;
    v.nbr = nbr;
    v.brp = brp.p;
    v.bcol = bcol.p;
    v.bval = bval.p;
    v.tp = tp.p;
    v.tk = tk.p;
    v.tb = tb.p;
    return v;
  }
};

struct Workspace {
  DBuf<int32_t> lo, hi, order, bin_cnt, bin_off;
  DBuf<int64_t> prod, bound, row_off, row_cnt, row_nnz, cnt, scan_tmp, l1r, l2r, i64tmp;
  DBuf<double> row_fsum, rs, partial, scal, passrow, row_p1;
  DBuf<int64_t> row_c1, cnt2;
  DBuf<int64_t> cursor;
  DBuf<int32_t> scr_col, pool_col;
  DBuf<double> scr_val, pool_val;
  DBuf<unsigned long long> pool_used;
  DBuf<int> row_counter, flags, fail_count, eqflag;
  DBuf<int32_t> fail_rows, fail_rows2;
  DBuf<int8_t> ident;
  DBuf<unsigned long long> prof;
  // BSR-8 views of the block kernels: B (the squared iterate or its halo rows; with its
  // block transpose) and A (a Taylor term's S^_{i-1}, no transpose)
  BsrBufs bsrB, bsrA;
  DBuf<int64_t> scan_tmp2;
  DBuf<double> bscr;
  int64_t pool_cap_hint = 0;
  // symmetric squaring (K3c / K3s / K3a): per block row |cand(I)|, |cand(I) >= I| and their
  // scans, the candidate lists and the upper output blocks
  DBuf<int64_t> sym_nj, sym_nup, sym_cjoff, sym_oboff;
  DBuf<int32_t> sym_cj, sym_wlo, sym_whi, sym_lidx;
  DBuf<unsigned long long> sym_bmask;
  DBuf<double> sym_fsI;
  DBuf<int64_t> sym_nzI, sym_rowcnt, sym_rowoff;
  DBuf<int64_t> fin_rowcnt, fin_sq, fin_l1I;
  DBuf<uint8_t> fin_flag;
  DBuf<double> fin_rsI, sym_psum;
  DBuf<double> sym_bstore;
  DBuf<int> sym_flag;
};

struct sexpm_plan_s {
  int dev = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  sexpm_options o{};
  int world = 1, rank = 0;
  std::unique_ptr<Transport> tr;  // world > 1
  int64_t n = 0, row_begin = 0, row_end = 0;
  std::vector<int64_t> bounds;  // world + 1 row bounds
  double eps_tol = 0.0;
  DCsr H0full;  // H0 = H 2^-N, all n rows (replicated)
  DCsr H0loc;   // this rank's rows of H0
  DCsr H0T;     // H0^T (CSC of H0, columns sorted by row) for the Taylor pull kernel
  // H0 as diagonals (when it has at most kDiaMax distinct offsets) for the Taylor push kernel
  int dia_nd = 0;
  int32_t dia_dmin = 0, dia_dmax = 0;
  DBuf<int32_t> dia_off;
  DBuf<double> dia_val;
  DBuf<unsigned long long> dia_prod;
  int dia_slots = 512;       // K5d accumulator slots per warp: adapted from the previous term's need
  bool dia_short_ok = true;  // the previous Taylor term's rows all fitted the short-row kernel K5s
  int dia_slots_max = 1152;  // the most that fit (set at plan time); retry size for rows over dia_slots
  DBuf<int> dia_need;
  std::vector<int32_t> h_dia_off;  // host copy of dia_off (descending)
  // K5w offset-window tables (build_window): U = the union of the Minkowski sums W_j of H0's
  // offsets, j = 1..M; lcnt[j] = |W_j|, ccnt[j] = |W_1 u ... u W_j| (ccnt[0] = 0)
  struct Win {
    bool ok = false;
    int nU = 0, dzero = -1, rw = 0;
    int64_t pad = 0, npad = 0;
    // half window (symmetric path): the terms are computed and stored over the offsets o >= 0
    // only (lcnt_h planes of stride plane = rows + padr, padr zero rows in front for the
    // mirrored reads of rows r + s, -padr <= s < 0); T^_0 over U_h; the FINAL tables map every
    // offset o of cum_m to |o| (row shift o < 0 ? o : 0)
    bool half = false;
    int nUh = 0;
    int64_t padr = 0;
    std::vector<int> lcnt_h;
    std::vector<int> lcnt, ccnt;      // |W_j|, |cum_j| (index j; ccnt[0] = 0)
    std::vector<int64_t> woff, coff;  // per term: start of its W-indexed / cum-indexed tables
    DBuf<int32_t> rec;                // TERM records (k_taylor_win), rw int32 per position
    DBuf<int16_t> neg1;               // -1 per cum position (FINAL when T^_0 is already complete)
    DBuf<int16_t> mapC, mapW, cumU;   // per cum position (T^_0 pass, FINAL): U-index if in the
                                      // previous cum (else -1), position in W_j (else -1), U-index
    DBuf<int32_t> coffs;
    DBuf<double> dpad;                // H0's diagonals zero-padded, plus a zero plane
    // T^_0 lives in place over U (position-major, plane u = offset U[u], plus a zero plane) in
    // the BSR view's value buffer, the S~ checkpoints in Tn.val and E.val: all three idle
    // until the squarings, so the Taylor phase maps no memory of its own
    DBuf<unsigned long long> cnt, need;
  } win;
  long long cache0[3] = {0, 0, 0};  // cache counters when the plan was created
  DCsr T, Tn, S, Sn, Bhalo, Ibuf, E;  // persistent (grow-only) iterates
  int32_t retries = 0;
  DBuf<int32_t> proc_order;  // K3 row processing order (cluster order of H's graph)
  // background computation of proc_order / group_start (overlaps the Taylor phase)
  std::thread bg;
  cudaStream_t bg_st = nullptr;
  cudaEvent_t ev_pattern = nullptr, ev_order = nullptr;
  bool order_pending = false;
  std::string bg_err;
  std::vector<int32_t> h_order, h_border;
  // squarings in aggregate order (option sq_order): perm[new] = old, 8-row aggregates of H's
  // graph; sq_tiled while the iterate is held in that order
  std::vector<int64_t> h_tperm;
  DBuf<int64_t> tperm, tinv;          // global maps (columns)
  DBuf<int64_t> tperm_loc, tinv_loc;  // this rank's rows (local indices)
  DBuf<int32_t> block_order_t;  // the aggregates (block rows in that order) in locality order
  bool sq_tiled = false;
  bool h_sym = false;   // H bit-exactly symmetric (plan time)
  bool t_index_pending = false;  // T^_0 kept in index order: the first squaring's BSR build relabels
  // the symmetric path hands the iterate between squarings on in block form: blk_out asks the
  // product for it (sym_finish_blocks writes ws.bsrB), blk_valid says ws.bsrB holds T^
  bool blk_out = false, blk_valid = false;
  int sq_index = 0;  // the squaring being computed (1..N; 0 in the Taylor phase)
  int64_t blk_nnz = 0;
  double blk_fmas = 0.0;
  bool sym_sq = false;  // this run squares on the symmetric path (option sym_squaring)
  int agg_kind = 0;  // 0 none, 1 BFS aggregates, 2 compact aggregates, 3 lattice diamonds, 4 lattice cubes
  bool tperm_ready = false;  // tperm / tinv (/ _loc) hold the squarings' aggregate relabelling
  double order_host_ms = 0.0, order_wait_ms = 0.0;  // background ordering thread: duration, wait
  DBuf<int32_t> block_order;  // block rows of the block kernel in locality order
  // H0's BSR-8 view in fragment order with its block transpose (Taylor terms on K3m), built
  // on first use; h0bsr_state 0 not built, 1 built, -1 not representable
  BsrBufs h0bsr;
  int h0bsr_state = 0;
  bool taylor_block = false;  // Taylor terms on K3m (K5d's accumulator overflowed)
  ~sexpm_plan_s() {
    if (bg.joinable()) bg.join();
    if (bg_st) cudaStreamSynchronize(bg_st);
    if (ev_pattern) cudaEventDestroy(ev_pattern);
    if (ev_order) cudaEventDestroy(ev_order);
    if (bg_st) cudaStreamDestroy(bg_st);
  }
  bool have_result = false;
  DBuf<double> apply_buf[2];  // sexpm_apply's intermediate steps
  // N3 reordering (option reorder = 1): perm[new] = old, inv[old] = new; H in RCM order
  DBuf<int64_t> perm, inv;
  DCsr Hperm, Etmp;
  int M = 0, N = 0, normal = 0, M_eff = 0;
  double norm = 0.0, a = 0.0, eps_g0 = 0.0;
  long double r0 = 0.0L;
  Workspace ws;
  sexpm_stats stats{};
  int sm_count = 148;
  size_t smem_per_sm = 233472;
  int numeric_blocks_per_sm = 2;
  int paged_blocks_per_sm = 3;
  float plan_ms = 0.f;
};

// ------------------------------------------------------------------------------------
// collectives on scalars: all-gather, then sum / max in rank order (identical everywhere)
// ------------------------------------------------------------------------------------
static void gather_doubles(sexpm_plan_s &P, const double *local, int cnt, std::vector<double> &all) {
  all.assign((size_t)cnt * P.world, 0.0);
  if (P.world == 1) {
    std::copy(local, local + cnt, all.begin());
    return;
  }
  DBuf<double> d;
  d.alloc((size_t)cnt * (P.world + 1), P.st);
  CK(cudaMemcpyAsync(d.p, local, cnt * sizeof(double), cudaMemcpyHostToDevice, P.st));
  P.tr->allgather(d.p, d.p + cnt, cnt * sizeof(double), P.st);
  CK(cudaMemcpyAsync(all.data(), d.p + cnt, (size_t)cnt * P.world * sizeof(double),
                     cudaMemcpyDeviceToHost, P.st));
  CK(cudaStreamSynchronize(P.st));
}
static double allsum(sexpm_plan_s &P, double v) {
  if (P.world == 1) return v;
  std::vector<double> all;
  gather_doubles(P, &v, 1, all);
  double s = 0.0;
  for (double x : all) s += x;
  return s;
}
static double allmax(sexpm_plan_s &P, double v) {
  if (P.world == 1) return v;
  std::vector<double> all;
  gather_doubles(P, &v, 1, all);
  double s = all[0];
  for (double x : all) s = std::max(s, x);
  return s;
}

template <typename T>
static T d2h(const T *dptr, cudaStream_t st) {
  T v;
  CK(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return v;
}

// B^T as CSR (= CSC of B) with every row sorted by column: count, scan, scatter, sort.
static void build_transpose(sexpm_plan_s &P, const CsrView &Bv, int64_t ncols, DCsr &BT) {
  cudaStream_t st = P.st;
  Workspace &w = P.ws;
  DBuf<int32_t> ccnt;
  ccnt.alloc((size_t)std::max<int64_t>(ncols, 1), st);
  CK(cudaMemsetAsync(ccnt.p, 0, ncols * sizeof(int32_t), st));
  launch_col_count(Bv, ccnt.p, st);
  DBuf<int64_t> cnt64, cursor;
  cnt64.alloc((size_t)std::max<int64_t>(ncols, 1), st);
  launch_i32_to_i64(ccnt.p, ncols, cnt64.p, st);
  BT.nrows = ncols;
  BT.row0 = 0;
  BT.nnz = Bv.nnz;
  BT.rp.alloc((size_t)ncols + 1, st);
  w.scan_tmp.ensure((size_t)scan_tmp_elems(ncols) + 1, st);
  launch_exclusive_scan(cnt64.p, ncols, BT.rp.p, w.scan_tmp.p, st);
  cursor.alloc((size_t)std::max<int64_t>(ncols, 1), st);
  CK(cudaMemcpyAsync(cursor.p, BT.rp.p, ncols * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  BT.col.alloc((size_t)std::max<int64_t>(Bv.nnz, 1), st);
  BT.val.alloc((size_t)std::max<int64_t>(Bv.nnz, 1), st);
  launch_transpose_fill(Bv, cursor.p, BT.col.p, BT.val.p, st);
  launch_sort_columns(ncols, BT.rp.p, BT.col.p, BT.val.p, st);
}

// ------------------------------------------------------------------------------------
// filtered product: C^ = Alg4.1((self*A + A*B)/div, eps_g)   [K1, K2, K3, K6, K4]
// A: local rows; B: rows covering every column of A.  C gets A's rows.
// ------------------------------------------------------------------------------------
// join the background order thread (once) and order the plan's stream after its upload
static void wait_order(sexpm_plan_s &P) {
  if (!P.order_pending) return;
  const auto w0 = std::chrono::steady_clock::now();
  if (P.bg.joinable()) P.bg.join();
  P.order_wait_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
  P.order_pending = false;
  REQUIRE(P.bg_err.empty(), SEXPM_ECUDA, P.bg_err);
  CK(cudaStreamWaitEvent(P.st, P.ev_order, 0));
}

// BSR-8 view of M's rows (block row I = rows 8I..8I+7 of the view; block columns global) in
// row-major (K3b) or fragment order (K3m), and its block transpose when asked.  Returns false
// (nothing built) when a block row spans more block columns than k_bsr_build's bitmap, or
// the view would not fit K3m's 32-bit block indices.
static void bsr_transpose(sexpm_plan_s &P, BsrBufs &b);
static bool build_bsr(sexpm_plan_s &P, const CsrView &M, bool frag, bool transpose, BsrBufs &b,
                      RowColMap map = RowColMap{}) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nbr = (M.nrows + 7) / 8, nbc = (P.n + 7) / 8;
  b.nbr = nbr;
  b.frag = frag;
  b.transposed = false;
  b.bcnt.ensure((size_t)nbr + 1, st);
  b.brp.ensure((size_t)nbr + 1, st);
  w.scan_tmp2.ensure((size_t)scan_tmp_elems(std::max(nbr, nbc)) + 1, st);
  CK(cudaMemsetAsync(w.flags.p, 0, sizeof(int), st));
  launch_bsr_count(M, nbr, b.bcnt.p, w.flags.p, st, map);
  launch_reduce_max_i64(b.bcnt.p, nbr, w.i64tmp.p + 7, st);
  launch_exclusive_scan(b.bcnt.p, nbr, b.brp.p, w.scan_tmp2.p, st);
  int bflags = 0;
  CK(cudaMemcpyAsync(&b.nb, b.brp.p + nbr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&b.bmax, w.i64tmp.p + 7, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&bflags, w.flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if ((bflags & 4) || (frag && b.nb >= (int64_t)INT32_MAX)) return false;
  const size_t nb1 = (size_t)std::max<int64_t>(b.nb, 1);
  b.bcol.ensure(nb1, st);
  b.bval.ensure(nb1 * 64, st);
  launch_bsr_fill(M, nbr, b.brp.p, b.bcol.p, b.bval.p, w.flags.p, st, frag, map);
  if (transpose) bsr_transpose(P, b);
  return true;
}

// the block transpose of a built view (column J's block rows K ascending, their block index)
static void bsr_transpose(sexpm_plan_s &P, BsrBufs &b) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nbr = b.nbr, nbc = (P.n + 7) / 8;
  const size_t nb1 = (size_t)std::max<int64_t>(b.nb, 1);
  {
    b.tcnt.ensure((size_t)nbc + 1, st);
    b.tp.ensure((size_t)nbc + 1, st);
    b.cnt64.ensure((size_t)nbc + 1, st);
    b.tk.ensure(nb1, st);
    b.tk_tmp.ensure(nb1, st);
    b.tb.ensure(nb1, st);
    b.tb_tmp.ensure(nb1, st);
    b.sort_tmp.ensure(bsr_transpose_temp_bytes(b.nb) + 256, st);
    b.keys_tmp.ensure(nb1, st);
    launch_bsr_transpose(nbr, nbc, b.nb, b.brp.p, b.bcol.p, b.tcnt.p, b.tp.p, b.tk_tmp.p, b.tb_tmp.p,
                         b.tk.p, b.tb.p, w.scan_tmp2.p, b.cnt64.p, b.sort_tmp.p, b.sort_tmp.n,
                         b.keys_tmp.p, st);
    b.transposed = true;
  }
}

// Algorithm 4.1: the scalar threshold recurrence on the host over the staged
// values of the rows (row_off / row_cnt / pool_val): F = sum of x^2 below the floor (dropped
// for sure), p1 = the first pass's sum when the product kernel fused it (tau_1 = eps_g).
// Returns the final threshold tau (keep |x| > tau) and the number of passes.
static double alg41_threshold(sexpm_plan_s &P, double eps_g, double F, bool fused_p1, double p1_local,
                              int64_t nr, int &passes, const SymOut *sym = nullptr, int64_t nbr = 0) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  passes = 0;
  if (eps_g == 0.0) return 0.0;  // reading R3: no filtering
  // m_0 = 1; the first pass always runs (reading R1, Theorem 4.1's proof P:384), then
  // the passes repeat while b_n > eps_g (1 + e_r)
  long double m = 1.0L, b = INFINITY;
  const long double eg = eps_g;
  const long double lim = eg * (1.0L + (long double)P.o.e_r);
  long double epsf = INFINITY;
  while (passes == 0 || b > lim) {
    epsf = eg / m;
    const double tau_d = (double)epsf;
    double S;
    if (passes == 0 && fused_p1 && tau_d == eps_g) {
      S = allsum(P, p1_local);  // tau_1 = eps_g: summed in the product kernel's flush
    } else {
      if (sym) {  // over the symmetric path's block store (per block row, rows in order)
        launch_sym_pass(*sym, nbr, tau_d, w.sym_psum.p, st);
        launch_reduce_sum(w.sym_psum.p, nbr, w.partial.p, w.scal.p + 1, st);
      } else {
        launch_alg41_pass_rows(nr, w.row_off.p, w.row_cnt.p, w.pool_val.p, tau_d, w.passrow.p,
                               w.partial.p, w.scal.p + 1, st);
      }
      S = allsum(P, d2h(w.scal.p + 1, st));
    }
    b = sqrtl((long double)F + (long double)S);
    m = b / epsf;
    passes++;
    REQUIRE(passes < 256, SEXPM_EINTERNAL, "Algorithm 4.1 pass cap reached (Theorem 4.1)");
  }
  return (double)epsf;
}

// The symmetric squaring stage (option sym_squaring; kernels.cuh SymOut): K3c counts, scans
// for the store layout, K3s products of the blocks J >= I, K3a rows.  Records k0 / k1 around
// K3s (rep.kernel_ms) and the K3c + K3a time in rep.asm_ms.  Returns false (nothing staged;
// the caller runs the full K3m) when a block row does not fit or the lists disagree.
static bool sym_squaring_stage(sexpm_plan_s &P, NumericArgs nh, const BsrView &Bv, int64_t nr,
                               bool long_lists, cudaEvent_t k0, cudaEvent_t k1, StepReport &rep,
                               double eps_g, double &floor_tau) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nbr = Bv.nbr;
  const size_t nb1 = (size_t)std::max<int64_t>(nbr, 1);
  w.sym_nj.ensure(nb1, st);
  w.sym_nup.ensure(nb1, st);
  w.sym_wlo.ensure(nb1, st);
  w.sym_whi.ensure(nb1, st);
  w.sym_cjoff.ensure(nb1 + 1, st);
  w.sym_oboff.ensure(nb1 + 1, st);
  w.sym_flag.ensure(1, st);
  w.scan_tmp2.ensure((size_t)scan_tmp_elems(nbr) + 1, st);
  cudaEvent_t c0, c1, a0, a1;
  CK(cudaEventCreate(&c0));
  CK(cudaEventCreate(&c1));
  CK(cudaEventCreate(&a0));
  CK(cudaEventCreate(&a1));
  CK(cudaEventRecord(c0, st));
  CK(cudaMemsetAsync(w.sym_flag.p, 0, sizeof(int), st));
  launch_sym_count(Bv, w.sym_nj.p, w.sym_nup.p, w.sym_wlo.p, w.sym_whi.p, w.sym_flag.p, st);
  if (d2h(w.sym_flag.p, st) & 32) {  // a block row's union wider than the small bitmaps
    CK(cudaMemsetAsync(w.sym_flag.p, 0, sizeof(int), st));
    launch_sym_count(Bv, w.sym_nj.p, w.sym_nup.p, w.sym_wlo.p, w.sym_whi.p, w.sym_flag.p, st, true);
  }
  launch_exclusive_scan(w.sym_nj.p, nbr, w.sym_cjoff.p, w.scan_tmp2.p, st);
  launch_exclusive_scan(w.sym_nup.p, nbr, w.sym_oboff.p, w.scan_tmp2.p, st);
  int64_t tot[2];
  int flag = 0;
  CK(cudaMemcpyAsync(&tot[0], w.sym_cjoff.p + nbr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&tot[1], w.sym_oboff.p + nbr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&flag, w.sym_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(c1, st));
  CK(cudaStreamSynchronize(st));
  bool ok = flag == 0 && tot[1] < ((int64_t)1 << 31);  // K3a's block indices are int32
  // test hook (tests/test_gpu_symmetric.py): SEXPM_SYM_FAIL = a bitmask of squarings (bit i-1 for
  // squaring i) whose symmetric product is refused, exercising the fall-backs
  if (const char *fe = getenv("SEXPM_SYM_FAIL"))
    if ((atoll(fe) >> (P.sq_index - 1)) & 1) ok = false;
  if (floor_tau == 0.0 && eps_g > 0.0) {
    // floor lemma: K = 64 x the candidate blocks of all block rows bounds the
    // number of entries of T~ (every nonzero lies in a candidate block)
    floor_tau = eps_g / sqrt(64.0 * (double)tot[0]);
  }
  nh.floor_tau = floor_tau;
  if (ok) {  // the stores must fit beside the live buffers (else: the full product)
    const double need = 8.0 * (double)tot[0] + 520.0 * (double)tot[1];
    std::lock_guard<std::mutex> lk(cache::mu);
    // what the stores already hold, or will reuse from the previous plan's parked buffers
    const double have_now = (double)(w.sym_cj.n * 4 + w.sym_lidx.n * 4 + w.sym_bmask.n * 8) +
                            (double)std::max<size_t>(w.sym_bstore.n * 8, w.sym_bstore.p ? 0 : cache::parked_bytes(w.sym_bstore.role)) +
                            (double)(w.sym_cj.p ? 0 : cache::parked_bytes(w.sym_cj.role));
    if (cache::budget == 0) {
      size_t fr = 0, tt = 0;
      cudaMemGetInfo(&fr, &tt);
      cache::budget = (size_t)(0.90 * (double)tt);
    }
    const double headroom = (double)cache::budget - (cache::bytes_allocated - cache::bytes_cached);
    if (need > have_now && 1.25 * need - have_now > 0.9 * headroom) ok = false;
  }
  if (ok) {
    w.sym_cj.ensure((size_t)std::max<int64_t>(tot[0], 1), st);
    w.sym_bstore.ensure((size_t)std::max<int64_t>(tot[1], 1) * 64, st);
    w.sym_lidx.ensure((size_t)std::max<int64_t>(tot[0], 1), st);
    SymOut so;
    so.bstore = w.sym_bstore.p;
    so.cj = w.sym_cj.p;
    so.ob_off = w.sym_oboff.p;
    so.cj_off = w.sym_cjoff.p;
    so.nj = w.sym_nj.p;
    so.nup = w.sym_nup.p;
    so.wlo = w.sym_wlo.p;
    w.sym_bmask.ensure((size_t)std::max<int64_t>(tot[1], 1), st);
    w.sym_fsI.ensure(nb1, st);
    w.sym_nzI.ensure(nb1, st);
    so.bmask = w.sym_bmask.p;
    so.fsI = w.sym_fsI.p;
    so.nzI = w.sym_nzI.p;
    w.sym_rowcnt.ensure((size_t)std::max<int64_t>(nr, 1), st);
    w.sym_rowoff.ensure((size_t)nr + 1, st);
    w.scan_tmp.ensure((size_t)scan_tmp_elems(nr) + 1, st);
    so.rowcnt = P.blk_out ? nullptr : w.sym_rowcnt.p;  // K3a's row counts: the last squaring
    so.lidx = w.sym_lidx.p;
    so.rowoff = w.sym_rowoff.p;
    if (!P.blk_out) CK(cudaMemsetAsync(w.sym_rowcnt.p, 0, (size_t)nr * sizeof(int64_t), st));
    so.whi = w.sym_whi.p;
    so.flag = w.sym_flag.p;
    CK(cudaMemsetAsync(w.row_counter.p, 0, sizeof(int), st));
    CK(cudaEventRecord(k0, st));
    launch_numeric_bsrm_sym(nh, Bv, nr, w.bscr.p, so, st, long_lists);
    CK(cudaEventRecord(k1, st));
    // the rows' pool offsets: a scan of K3s's kept counts (deterministic layout)
    CK(cudaEventRecord(a0, st));
    int64_t total = 0;
    if (!P.blk_out) {  // (handed on in block form: no rows are staged)
      launch_exclusive_scan(w.sym_rowcnt.p, nr, w.sym_rowoff.p, w.scan_tmp.p, st);
      CK(cudaMemcpyAsync(&total, w.sym_rowoff.p + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(&flag, w.sym_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ok = flag == 0;
    if (ok && total > nh.pool_cap) {  // exact size known: grow the pool, no re-run
      w.pool_col.ensure((size_t)total, st);
      w.pool_val.ensure((size_t)total, st);
      nh.pool_col = w.pool_col.p;
      nh.pool_val = w.pool_val.p;
      nh.pool_cap = (int64_t)std::min(w.pool_col.n, w.pool_val.n);
    }
    if (ok) {  // K3a only over K3s's complete lists
      if (!P.blk_out)
        CK(cudaMemcpyAsync(w.pool_used.p, w.sym_rowoff.p + nr, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      launch_sym_lidx(so, nbr, st);
      if (!P.blk_out) launch_sym_assemble(nh, so, nbr, nr, P.sm_count * 4, st);
      CK(cudaEventRecord(a1, st));
      CK(cudaMemcpyAsync(&flag, w.sym_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ok = flag == 0;
      float ms_c = 0.f, ms_a = 0.f;
      CK(cudaEventElapsedTime(&ms_c, c0, c1));
      CK(cudaEventElapsedTime(&ms_a, a0, a1));
      rep.asm_ms = ms_c + ms_a;
    }
  }
  if (!ok) {
    if (getenv("SEXPM_STEP_LOG"))
      fprintf(stderr, "[sexpm run] symmetric squaring handed to the full product (flag %d)\n", flag);
    CK(cudaMemsetAsync(w.pool_used.p, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(w.flags.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(w.row_counter.p, 0, sizeof(int), st));  // K3s consumed the scheduler
    CK(cudaEventRecord(k0, st));
  }
  for (cudaEvent_t e : {c0, c1, a0, a1}) cudaEventDestroy(e);
  return ok;
}

static SymOut sym_out_of(Workspace &w) {
  SymOut so;
  so.bstore = w.sym_bstore.p;
  so.bmask = w.sym_bmask.p;
  so.fsI = w.sym_fsI.p;
  so.nzI = w.sym_nzI.p;
  so.cj = w.sym_cj.p;
  so.ob_off = w.sym_oboff.p;
  so.cj_off = w.sym_cjoff.p;
  so.nj = w.sym_nj.p;
  so.nup = w.sym_nup.p;
  so.wlo = w.sym_wlo.p;
  so.whi = w.sym_whi.p;
  so.flag = w.sym_flag.p;
  so.rowcnt = w.sym_rowcnt.p;
  so.rowoff = w.sym_rowoff.p;
  so.lidx = w.sym_lidx.p;
  return so;
}

static int64_t so_nup_total(Workspace &w, int64_t nbr, cudaStream_t st) {
  return d2h(w.sym_oboff.p + nbr, st);  // the scan of K3c's upper counts
}

// The symmetric product's result handed on in block form (no staging, no CSR): Algorithm 4.1
// over the block store (passes k_sym_pass), then the next squaring's BSR-8 view written from
// the store with |x| > tau into ws.bsrB (k_sym_fin count / scan / write), with the iterate's
// statistics (nnz, ||I + T^||_F, bandwidths, and sum_r nnz_r^2 + nnz: the next product count)
static void sym_finish_blocks(sexpm_plan_s &P, double eps_g, int64_t nr, StepReport &rep) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nbr = (nr + 7) / 8;
  const size_t nb1 = (size_t)std::max<int64_t>(nbr, 1);
  const SymOut so = sym_out_of(w);
  w.sym_psum.ensure(nb1, st);
  launch_reduce_sum(w.sym_fsI.p, nbr, w.partial.p, w.scal.p + 0, st);
  launch_reduce_sum_i64(w.sym_nzI.p, nbr, w.i64tmp.p + 3, st);
  CK(cudaMemsetAsync(w.i64tmp.p + 4, 0, sizeof(int64_t), st));  // (no rows staged)
  double F = 0.0;
  int64_t hz[2];
  CK(cudaMemcpyAsync(&F, w.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hz, w.i64tmp.p + 3, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  rep.nnz_unf = hz[0];
  rep.staged = hz[1];
  rep.fsum = F;
  int passes = 0;
  const double tau = alg41_threshold(P, eps_g, F, false, 0.0, nr, passes, &so, nbr);
  rep.passes = passes;
  rep.tau = tau;
  // the next view: counts and statistics, scan, blocks
  BsrBufs &b = w.bsrB;
  b.nbr = nbr;
  b.frag = true;
  b.transposed = false;
  b.bcnt.ensure(nb1 + 1, st);
  b.brp.ensure(nb1 + 1, st);
  const size_t nr1 = (size_t)std::max<int64_t>(nr, 1);
  w.fin_rowcnt.ensure(nr1, st);
  w.fin_sq.ensure(nr1, st);
  w.fin_flag.ensure((size_t)std::max<int64_t>(so_nup_total(w, nbr, st), 1), st);
  w.fin_l1I.ensure(nb1, st);
  w.fin_rsI.ensure(nb1, st);
  w.scan_tmp2.ensure((size_t)scan_tmp_elems(std::max<int64_t>(nbr, nr)) + 1, st);
  CK(cudaMemsetAsync(b.bcnt.p, 0, nb1 * sizeof(int64_t), st));
  CK(cudaMemsetAsync(w.fin_rowcnt.p, 0, nr1 * sizeof(int64_t), st));
  SymFin f;
  f.bcnt = b.bcnt.p;
  f.rowcnt = w.fin_rowcnt.p;
  f.flag = w.fin_flag.p;
  f.rsI = w.fin_rsI.p;
  f.l1I = w.fin_l1I.p;
  launch_sym_fin(so, nbr, nr, tau, f, false, st);
  launch_exclusive_scan(b.bcnt.p, nbr, b.brp.p, w.scan_tmp2.p, st);
  launch_rowcnt_sq(w.fin_rowcnt.p, nr, w.fin_sq.p, st);
  launch_reduce_sum_i64(w.fin_rowcnt.p, nr, w.i64tmp.p + 0, st);
  launch_reduce_sum_i64(w.fin_sq.p, nr, w.i64tmp.p + 1, st);
  launch_reduce_max_i64(w.fin_l1I.p, nbr, w.i64tmp.p + 2, st);
  launch_reduce_max_i64(b.bcnt.p, nbr, w.i64tmp.p + 6, st);
  launch_reduce_sum(w.fin_rsI.p, nbr, w.partial.p, w.scal.p + 2, st);
  int64_t hs[7];
  double rs = 0.0;
  CK(cudaMemcpyAsync(hs, w.i64tmp.p, 7 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rs, w.scal.p + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&b.nb, b.brp.p + nbr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  b.bmax = hs[6];
  const size_t nbb = (size_t)std::max<int64_t>(b.nb, 1);
  b.bcol.ensure(nbb, st);
  b.bval.ensure(nbb * 64, st);
  f.brp = b.brp.p;
  f.bcol = b.bcol.p;
  f.bval = b.bval.p;
  launch_sym_fin(so, nbr, nr, tau, f, true, st);
  CK(cudaGetLastError());
  rep.nnz = hs[0];
  rep.normIT2 = rs;
  rep.l1 = hs[2];
  rep.l2 = hs[2];  // symmetric
  P.blk_valid = true;
  P.blk_nnz = hs[0];
  P.blk_fmas = (double)hs[1] + (double)hs[0];  // sum_k nnz(row k)^2 + nnz (the 2T term)
}

static void filtered_product(sexpm_plan_s &P, const CsrView &A, const CsrView &B, double self,
                            double div, double eps_g, DCsr &C, StepReport &rep,
                            const DCsr *BT = nullptr, bool add_identity = false,
                            const DCsr *acc = nullptr, DCsr *acc_out = nullptr) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nr = A.nrows;
  const int okern = P.o.kernel == 8 ? 0 : P.o.kernel;  // 8: the window kernel (Taylor phase)
  const size_t nr1 = (size_t)std::max<int64_t>(nr, 1);
  w.lo.ensure(nr1, st);
  w.hi.ensure(nr1, st);
  w.order.ensure(nr1, st);
  w.prod.ensure(nr1, st);
  w.bound.ensure(nr1, st);
  w.row_off.ensure(nr1, st);
  w.row_cnt.ensure(nr1, st);
  w.row_nnz.ensure(nr1, st);
  w.row_fsum.ensure(nr1, st);
  w.passrow.ensure(nr1, st);
  w.cnt.ensure(nr1, st);
  w.rs.ensure(nr1, st);
  w.l1r.ensure(nr1, st);
  w.l2r.ensure(nr1, st);
  w.scan_tmp.ensure((size_t)scan_tmp_elems(nr) + 1, st);
  w.bin_cnt.ensure(64, st);
  w.bin_off.ensure(64, st);
  w.partial.ensure(1024, st);
  w.scal.ensure(8, st);
  w.i64tmp.ensure(8, st);
  w.pool_used.ensure(1, st);
  w.row_counter.ensure(1, st);
  w.flags.ensure(1, st);

  // Taylor term with a diagonal H0: the push kernel K5d needs no symbolic pass; every
  // product count is bounded by ndiag * nnz(A), a valid K for the floor lemma
  const bool dia_path = self == 0.0 && P.dia_nd > 0 && B.rp == P.H0full.rp.p &&
                        (okern == 0 || okern == 7);
  // a squaring (of T^, or of E in the SSAT baseline): A and B are the same matrix (or B its
  // halo rows), with or without the 2T term
  const bool sq_like = self != 0.0 || B.rp == A.rp || (P.Bhalo.rp.p && B.rp == P.Bhalo.rp.p);
  int64_t hstat[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool have_symbolic = false;
  auto run_symbolic = [&]() {  // K1 symbolic bounds
    launch_symbolic(A, B, self != 0.0 ? 1 : 0, w.lo.p, w.hi.p, w.prod.p, w.bound.p, st);
    launch_reduce_sum_i64(w.bound.p, nr, w.i64tmp.p + 0, st);
    launch_reduce_max_i64(w.bound.p, nr, w.i64tmp.p + 1, st);
    launch_reduce_sum_i64(w.prod.p, nr, w.i64tmp.p + 2, st);
    // longest A row (cursor scratch size)
    launch_row_lengths(A.rp, nr, w.cnt.p, st);
    launch_reduce_max_i64(w.cnt.p, nr, w.i64tmp.p + 6, st);
    CK(cudaMemcpyAsync(hstat, w.i64tmp.p, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    have_symbolic = true;
  };
  double Kglob;
  // the symmetric squaring needs no K1: its K (floor lemma) is K3c's candidate-slot count and
  // its products follow from the row lengths (symmetric pattern: sum_k nnz(row k)^2)
  const bool sym_planned = P.sym_sq && self == 2.0 && B.rp == A.rp && nr == P.n && A.row0 == 0 &&
                           (okern == 0 || okern == 13) && !P.o.exact_products;
  if (dia_path) {
    hstat[0] = (int64_t)P.dia_nd * A.nnz;
    Kglob = allsum(P, (double)hstat[0]);
  } else if (sym_planned && P.blk_valid) {  // the iterate in block form (sym_finish_blocks)
    hstat[2] = (int64_t)P.blk_fmas;
    hstat[0] = (int64_t)1 << 60;
    Kglob = 0.0;
  } else if (sym_planned) {
    launch_rowlen_sq(A.rp, nr, w.bound.p, st);
    launch_reduce_sum_i64(w.bound.p, nr, w.i64tmp.p + 2, st);
    hstat[2] = d2h(w.i64tmp.p + 2, st) + A.nnz;
    hstat[0] = (int64_t)1 << 60;  // no bound on the staging pool (K3a's total is exact)
    Kglob = 0.0;                  // set by the stage from K3c
  } else {
    run_symbolic();
    Kglob = allsum(P, (double)hstat[0]);
  }
  rep.fmas = (double)hstat[2];
  double floor_tau = (eps_g > 0.0 && Kglob > 0.0) ? eps_g / sqrt(Kglob) : 0.0;

  // K2 scheduling order: the plan's locality (cluster) order when it covers these rows,
  // else longest-processing-time-first bins
  // the locality order serves the squarings (Taylor terms stream their rows in index order)
  const bool use_cluster = sq_like && !P.sq_tiled && P.proc_order.p && (int64_t)P.proc_order.n >= nr &&
                           A.row0 == P.row_begin && nr == P.row_end - P.row_begin;
  if (use_cluster) wait_order(P);
  // the block kernels schedule block rows themselves: row bins only for the row kernels
  const bool block_sq = sq_like && (okern == 0 || okern == 11 || okern == 13);
  const bool binned = !use_cluster && have_symbolic && !block_sq;
  if (binned) launch_bin_rows(nr, w.prod.p, w.bin_cnt.p, w.bin_off.p, w.order.p, st);

  // K3 numeric
  NumericArgs na;
  na.A = A;
  na.B = B;
  na.self_coef = self;
  na.divisor = div;
  na.floor_tau = floor_tau;
  na.lo = w.lo.p;
  na.hi = w.hi.p;
  na.order = use_cluster ? P.proc_order.p : (binned ? w.order.p : nullptr);
  na.window = P.o.window_cols > 0 ? P.o.window_cols : 8192;
  na.grid = (int)std::max<int64_t>(1, std::min<int64_t>(nr, (int64_t)P.sm_count * P.numeric_blocks_per_sm));
  na.cursor_cap = std::max<int64_t>(hstat[6], 1);
  na.scr_cap = std::max<int64_t>(hstat[1], 1);
  int64_t cap = std::max<int64_t>(w.pool_cap_hint, (sq_like ? 3 : 2) * A.nnz + 2 * nr + 1024);
  double sum_bound = 0;  // exact upper bound
  sum_bound = (double)hstat[0];
  if ((double)cap > sum_bound) cap = (int64_t)sum_bound + 1;
  cudaEvent_t e0, e1, e_first;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e_first));
  bool have_first = false;
  unsigned long long used = 0;
  bool fused_p1 = false;
  w.row_p1.ensure(nr1, st);
  w.row_c1.ensure(nr1, st);
  w.fail_rows.ensure(nr1, st);
  w.fail_rows2.ensure(nr1, st);
  w.fail_count.ensure(1, st);
  const int paged_grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(nr, (int64_t)P.sm_count * P.paged_blocks_per_sm));
  int nfail_other = 0;  // rows finished by kernels other than the first (and its K5d retry)
  bool dia_launched = false;
  bool sym_failed = false;  // the symmetric path could not hold this product: full K3m
  for (int attempt = 0;; attempt++) {
    nfail_other = 0;
    w.pool_col.ensure((size_t)cap, st);
    w.pool_val.ensure((size_t)cap, st);
    na.pool_col = w.pool_col.p;
    na.pool_val = w.pool_val.p;
    na.pool_cap = (int64_t)std::min(w.pool_col.n, w.pool_val.n);
    na.pool_used = w.pool_used.p;
    na.row_off = w.row_off.p;
    na.row_cnt = w.row_cnt.p;
    na.row_fsum = w.row_fsum.p;
    na.row_nnz = w.row_nnz.p;
    na.row_counter = w.row_counter.p;
    na.flags = w.flags.p;
    CK(cudaMemsetAsync(w.pool_used.p, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(w.row_counter.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(w.flags.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(w.fail_count.p, 0, sizeof(int), st));
    CK(cudaEventRecord(e0, st));
    int kern = okern;
    const bool taylor_pull_ok = self == 0.0 && BT != nullptr && BT->rp.p != nullptr;
    // squarings: the block kernel on the fp64 tensor-core instruction (13; 11 is the
    // bit-exact DMUL/DADD variant); Taylor terms: the diagonal push or the pull kernel
    // (Taylor terms whose rows outgrew K5d's accumulator -- 3D stencils -- go to the
    // tensor-core block kernel with B = H0)
    if (kern == 0) {
      if (sq_like) kern = P.o.exact_products ? 11 : 13;
      else if (P.taylor_block) kern = 13;
      else kern = dia_path ? 7 : (taylor_pull_ok ? 6 : 5);
    }
    // the exact block kernel squares one matrix (or a rank's rows inside its halo rows)
    if (kern == 11 && !sq_like) kern = dia_path ? 7 : (taylor_pull_ok ? 6 : 5);
    // the block kernel needs B's rows block-aligned and A's rows a block-aligned slice of them
    // (one GPU: A = B; several: A = the rank's rows inside its halo B, 8-aligned partition)
    const bool same = B.rp == A.rp;
    bool bsr_ok = same;
    if (!same && (kern == 11 || kern == 13) && B.row0 % 8 == 0 && A.row0 >= B.row0 &&
        (A.row0 - B.row0) % 8 == 0 && A.row0 + nr <= B.row0 + B.nrows) {
      // A must be a slice of B (the rank's rows inside its halo): checked, not assumed
      w.eqflag.ensure(1, st);
      CK(cudaMemsetAsync(w.eqflag.p, 0, sizeof(int), st));
      launch_rows_equal(A, B, w.eqflag.p, st);
      bsr_ok = d2h(w.eqflag.p, st) == 0;
    }
    if (sq_like && (kern == 11 || kern == 13) && !bsr_ok) kern = 5;
    if (kern == 7 && !dia_path) kern = taylor_pull_ok ? 6 : 5;
    if (kern == 6 && !taylor_pull_ok) kern = 5;
    if (kern == 7) CK(cudaMemsetAsync(P.dia_prod.p, 0, sizeof(unsigned long long), st));
    int nfail = 0;
    {
      // staged chain: the chosen shared-memory kernel over all rows, rows it cannot hold
      // go to the next one (pull -> hash -> block window; paged / k-sync / hash -> window)
      const int32_t *list = na.order;
      int64_t nlist = nr;
      int32_t *fbuf[2] = {w.fail_rows.p, w.fail_rows2.p};
      int fb = 0;
      int stage = kern;
      bool first = true, dia_retry = false;
      // short rows first (thread-per-row K5s) while the previous term's rows were short
      bool dia_short = P.dia_short_ok;
      // the paged (5) and diagonal (7) kernels fuse Algorithm 4.1's first pass into their flush
      fused_p1 = eps_g > 0.0 && (kern == 5 || kern == 7 || kern == 11 || kern == 13);
      while (nlist > 0) {
        if (stage != 7 && !have_symbolic && !(sym_planned && stage == 13 && !sym_failed)) {
          // rows left by K5d: the other kernels need K1 (the symmetric squaring does not)
          run_symbolic();
          rep.fmas = (double)hstat[2];
          na.cursor_cap = std::max<int64_t>(hstat[6], 1);
          na.scr_cap = std::max<int64_t>(hstat[1], 1);
        }
        NumericArgs nh = na;
        nh.order = list;
        nh.nlist = nlist;
        if ((first || stage == 7) && fused_p1) {
          nh.row_p1 = w.row_p1.p;
          nh.row_c1 = w.row_c1.p;
          nh.eps_g = eps_g;
        }
        CK(cudaMemsetAsync(w.row_counter.p, 0, sizeof(int), st));
        CK(cudaMemsetAsync(w.fail_count.p, 0, sizeof(int), st));
        if (stage == 3) {
          w.cursor.ensure((size_t)na.grid * na.cursor_cap, st);
          w.scr_col.ensure((size_t)na.grid * na.scr_cap, st);
          w.scr_val.ensure((size_t)na.grid * na.scr_cap, st);
          nh.cursor = w.cursor.p;
          nh.scr_col = w.scr_col.p;
          nh.scr_val = w.scr_val.p;
          nh.grid = (int)std::min<int64_t>(na.grid, nlist);
          launch_numeric(nh, st);
          CK(cudaGetLastError());
          break;
        }
        int32_t *fout = fbuf[fb];
        if (stage == 5) {
          nh.grid = paged_grid;
          launch_numeric_paged(nh, fout, w.fail_count.p, st);
        } else if (stage == 11 || stage == 13) {
          // BSR-8 view of B (= A, or A's halo rows; for a Taylor term H0, built once per plan)
          // with its block transpose, A's own view for a Taylor term, then the block kernel
          // over A's block rows
          const int64_t nbr_a = (nr + 7) / 8;
          const bool taylor = !sq_like;
          bool ok_view;
          bool sym_try = false;
          if (taylor && B.rp != P.H0full.rp.p) {
            ok_view = false;  // a product with any other B: its view is not kept
          } else if (taylor) {
            if (P.h0bsr_state == 0)
              P.h0bsr_state = build_bsr(P, P.H0full.view(), true, true, P.h0bsr) ? 1 : -1;
            ok_view = P.h0bsr_state == 1 && build_bsr(P, A, true, false, w.bsrA);
          } else {
            // the symmetric kernel reads B_KJ as B_JK^T: no block transpose (built on fallback)
            sym_try = stage == 13 && P.sym_sq && same && nr == P.n && self == 2.0 && !sym_failed;
            // T^_0 still in index order (do_run): the relabelling into aggregates fused here
            RowColMap map;
            if (P.t_index_pending && sym_try) {
              map.rowmap = P.tperm_loc.p;
              map.colmap = P.tinv.p;
            }
            if ((P.t_index_pending || P.blk_valid) && !sym_try) {  // only the symmetric path takes it
              rep.relabel_needed = P.t_index_pending;
              rep.need_csr = P.blk_valid;
              cudaEventDestroy(e0);
              cudaEventDestroy(e1);
              cudaEventDestroy(e_first);
              return;
            }
            ok_view = P.blk_valid ? true : build_bsr(P, B, stage == 13, !sym_try, w.bsrB, map);
            // K3b holds a row of A in shared memory
            if (ok_view && stage == 11 && w.bsrB.bmax > kBsrMaxRowBlocks) ok_view = false;
          }
          if (!ok_view) {  // the whole product goes to the paged kernel
            stage = 5;
            continue;
          }
          const BsrBufs &bb = taylor ? P.h0bsr : w.bsrB;
          const int64_t nb = bb.nb;
          BsrView Bv = bb.view();
          if (taylor) {
            Bv.abrp = w.bsrA.brp.p;
            Bv.abcol = w.bsrA.bcol.p;
            Bv.abval = w.bsrA.bval.p;
          }
          Bv.nbr_a = nbr_a;
          Bv.ib0 = taylor ? 0 : (A.row0 - B.row0) / 8;
          Bv.kb0 = B.row0 / 8;
          if (use_cluster && nr == P.row_end - P.row_begin && A.row0 % 8 == 0 && !getenv("SEXPM_BSR_NATURAL"))
            Bv.border = P.block_order.p;  // block rows of the rank's rows in locality order
          if (P.sq_tiled && same && nr == P.n && !getenv("SEXPM_BSR_NATURAL"))
            Bv.border = P.block_order_t.p;  // the aggregates in locality order
          // long match lists (3D): fewer, deeper-pipelined warps
          const BsrBufs &av = taylor ? w.bsrA : w.bsrB;
          const bool long_lists = av.nbr > 0 && av.nb > (int64_t)kBsrMLongRow * av.nbr;
          nh.grid = (int)std::max<int64_t>(
              1, std::min<int64_t>(nbr_a, (int64_t)P.sm_count * (stage == 13 ? (long_lists ? kBsrMBlocksPerSmLong : kBsrMBlocksPerSm) : 2)));
          w.bscr.ensure((size_t)nh.grid * (stage == 13 ? (size_t)kBsrMJCap * 66 : (size_t)kBsrScratchPerCta), st);
          CK(cudaMemsetAsync(w.row_counter.p, 0, sizeof(int), st));
          w.prof.ensure(16, st);
          CK(cudaMemsetAsync(w.prof.p, 0, 16 * sizeof(unsigned long long), st));
          nh.prof = w.prof.p;
          cudaEvent_t k0, k1;  // the block kernel alone (the stage also builds the view)
          CK(cudaEventCreate(&k0));
          CK(cudaEventCreate(&k1));
          CK(cudaEventRecord(k0, st));
          // symmetric squaring: one GPU, T exactly symmetric (do_run), A = B
          bool sym_done = false;
          if (sym_try) {
            sym_done = sym_squaring_stage(P, nh, Bv, nr, long_lists, k0, k1, rep, eps_g, floor_tau);
            rep.sym = sym_done;
            if (!sym_done && (P.t_index_pending || P.blk_valid)) {  // do_run re-runs on the CSR
              rep.relabel_needed = P.t_index_pending;
              rep.need_csr = P.blk_valid;
              cudaEventDestroy(k0);
              cudaEventDestroy(k1);
              cudaEventDestroy(e0);
              cudaEventDestroy(e1);
              cudaEventDestroy(e_first);
              return;
            }
            if (!sym_done) {  // the full K3m: it needs the block transpose and K1's spans
              sym_failed = true;
              if (!have_symbolic) {
                run_symbolic();
                nh.lo = w.lo.p;
                nh.hi = w.hi.p;
              }
              nh.floor_tau = floor_tau;
              bsr_transpose(P, w.bsrB);
              Bv.tp = w.bsrB.tp.p;
              Bv.tk = w.bsrB.tk.p;
              Bv.tb = w.bsrB.tb.p;
              CK(cudaEventRecord(k0, st));
            }
          }
          if (sym_done) {
            // K3s + K3a staged every row
          } else if (stage == 13)
            launch_numeric_bsrm(nh, Bv, nr, w.bscr.p, fout, w.fail_count.p, st, long_lists);
          else
            launch_numeric_bsr(nh, Bv, nr, w.bscr.p, fout, w.fail_count.p, st);
          if (!sym_done) CK(cudaEventRecord(k1, st));
          CK(cudaEventSynchronize(k1));
          CK(cudaEventElapsedTime(&rep.kernel_ms, k0, k1));
          cudaEventDestroy(k0);
          cudaEventDestroy(k1);
          rep.bsr_blocks = nb;
          unsigned long long nbp = 0;
          CK(cudaMemcpy(&nbp, w.prof.p, sizeof(nbp), cudaMemcpyDeviceToHost));
          rep.block_products = (double)nbp;
          if (getenv("SEXPM_STEP_LOG")) {
            unsigned long long pr[5];
            CK(cudaMemcpy(pr, w.prof.p, sizeof(pr), cudaMemcpyDeviceToHost));
            fprintf(stderr, "[sexpm run] block kernel %d: block rows handed on: K span %llu, J span %llu, both %llu, J count %llu\n",
                    stage, pr[1], pr[2], pr[3], pr[4]);
          }
        } else if (stage == 7) {
          DiaView D;
          D.ndiag = P.dia_nd;
          D.off = P.dia_off.p;
          D.val = P.dia_val.p;
          D.n = P.n;
          D.dmin = P.dia_dmin;
          D.dmax = P.dia_dmax;
          D.prod_count = P.dia_prod.p;
          // slots sized from the previous term's largest row (occupancy: 20 -> 28+ warps/SM
          // at config 5); rows over it are retried once at twice the slots
          if (dia_short) {
            launch_taylor_dia_short(nh, D, fout, w.fail_count.p, st);
          } else {
          const int slots = std::min(dia_retry ? 2 * P.dia_slots : P.dia_slots, P.dia_slots_max);
          if (!dia_retry) CK(cudaMemsetAsync(P.dia_need.p, 0, sizeof(int), st));
          D.need_max = P.dia_need.p;
          const int per_sm = std::max(1, std::min(16, (int)(P.smem_per_sm / (taylor_dia_smem_bytes(slots) + 1024))));
          nh.grid = (int)std::max<int64_t>(1, std::min<int64_t>((nlist + kDiaWarpsPerCta - 1) / kDiaWarpsPerCta,
                                                                (int64_t)P.sm_count * per_sm));
          launch_taylor_dia(nh, D, slots, fout, w.fail_count.p, st);
          dia_launched = true;
          }
        } else {  // 6
          nh.grid = paged_grid;
          launch_taylor_pull(nh, BT->view(), fout, w.fail_count.p, st);
        }
        CK(cudaGetLastError());
        if (first) {
          CK(cudaEventRecord(e_first, st));
          first = false;
          have_first = true;
        }
        const int nf = d2h(w.fail_count.p, st);
        nfail += nf;
        list = fout;
        nlist = nf;
        fb ^= 1;
        // fall-through: K5d rows over its slots -> K5d at twice the slots -> paged; K5p ->
        // hash; the squaring kernels -> paged; everything else -> the block-window kernel (no
        // capacity limit)
        if (stage == 7 && dia_short) {
          dia_short = false;  // rows wider than K5s's window: the warp kernel K5d
        } else if (stage == 7 && !dia_retry && P.dia_slots < P.dia_slots_max) {
          dia_retry = true;
        } else {
          stage = (stage == 7 || stage == 6 || stage == 11 || stage == 13) ? 5 : 3;
          nfail_other += nf;
        }
      }
    }
    rep.window_rows = nfail;
    if (nfail_other > 0) fused_p1 = false;  // rows handled by kernels without the fused pass
    CK(cudaEventRecord(e1, st));
    int flags = 0;
    CK(cudaMemcpyAsync(&flags, w.flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&used, w.pool_used.p, sizeof(used), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    REQUIRE(!(flags & 2), SEXPM_EINTERNAL, "numeric: per-CTA staging overflow");
    if (!(flags & 1)) break;
    REQUIRE(attempt < 8, SEXPM_EINTERNAL, "numeric: staging pool keeps overflowing");
    cap = std::max<int64_t>(2 * cap, (int64_t)(1.25 * (double)used) + 1024);
    P.retries++;
  }
  CK(cudaEventElapsedTime(&rep.numeric_ms, e0, e1));
  rep.first_ms = rep.numeric_ms;
  if (have_first) CK(cudaEventElapsedTime(&rep.first_ms, e0, e_first));
  cudaEventDestroy(e_first);
  if (dia_path && !have_symbolic && nfail_other == 0) rep.fmas = (double)d2h(P.dia_prod.p, st);
  if (dia_path) P.dia_short_ok = !dia_launched;  // next term: K5s first only if every row fitted it
  if (dia_launched) {  // next term's K5d slots: this term's largest row + 12.5 % + 64, 64-aligned
    const long long nd = d2h(P.dia_need.p, st);
    P.dia_slots = (int)std::min<long long>(P.dia_slots_max, std::max<long long>(256, ((nd * 9 / 8 + 64 + 63) / 64) * 64));
    // rows beyond K5d's largest accumulator went to the paged kernel: the next terms run on
    // the tensor-core block kernel (B = H0) instead
    // (also once rows needed over half of it, or > 1 % of the rows were retried or handed on:
    // 3D rows keep growing term after term)
    if (okern == 0 && !P.o.exact_products && (nd > P.dia_slots_max / 2 || rep.window_rows * 100 > nr))
      P.taylor_block = true;
    if (getenv("SEXPM_STEP_LOG")) fprintf(stderr, "[sexpm run] K5d need %lld slots, next %d (max %d), retried rows %d\n", nd, P.dia_slots, P.dia_slots_max, (int)(rep.window_rows - nfail_other));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  w.pool_cap_hint = std::max<int64_t>(w.pool_cap_hint, (int64_t)(1.2 * (double)used));
  rep.staged = (int64_t)used;
  // compulsory bytes of K3: A (rowptr + entries), the B rows it reads (whole B: each row once;
  // when B is A itself it is read once), staged writes (col + val) and per-row outputs.
  {
    const bool same = (B.rp == A.rp);
    rep.numeric_bytes = 8.0 * (nr + 1) + 12.0 * (double)A.nnz +
                        (same ? 0.0 : 8.0 * (B.nrows + 1) + 12.0 * (double)B.nnz) +
                        12.0 * (double)used + 32.0 * (double)nr;
  }

  if (rep.sym && P.blk_out) {  // handed on in block form: no staging, no CSR
    P.blk_valid = false;       // the input view is consumed; sym_finish_blocks writes the next
    sym_finish_blocks(P, eps_g, nr, rep);
    return;
  }
  P.blk_valid = false;
  // Algorithm 4.1: scalar recurrence on the host, sums on the device (one
  // read-back for the floor sum, the distinct count and the fused first pass)
  launch_reduce_sum(w.row_fsum.p, nr, w.partial.p, w.scal.p + 0, st);
  launch_reduce_sum_i64(w.row_nnz.p, nr, w.i64tmp.p + 3, st);
  if (fused_p1) launch_reduce_sum(w.row_p1.p, nr, w.partial.p, w.scal.p + 3, st);
  double hs[4];
  int64_t hnz = 0;
  CK(cudaMemcpyAsync(hs, w.scal.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hnz, w.i64tmp.p + 3, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double Floc = hs[0];
  rep.nnz_unf = (int64_t)allsum(P, (double)hnz);
  const double F = allsum(P, Floc);
  rep.fsum = F;
  int passes = 0;
  const double tau = alg41_threshold(P, eps_g, F, fused_p1, fused_p1 ? hs[3] : 0.0, nr, passes);
  rep.passes = passes;
  rep.tau = tau;

  // K4 compaction + fused row statistics (+ E = I + T^_N on the last squaring)
  if (add_identity) {
    w.ident.ensure(nr1, st);
    launch_compact_count_ident(nr, A.row0, w.row_off.p, w.row_cnt.p, w.pool_col.p, w.pool_val.p,
                               tau, w.cnt.p, w.ident.p, st);
    launch_count_ident(w.ident.p, nr, w.i64tmp.p + 6, st);
  } else if (fused_p1 && passes == 1 && tau == eps_g) {
    launch_copy_i64_offset(w.row_c1.p, nr, 0, w.cnt.p, st);  // kept = staged |x| > eps_g
  } else {
    launch_compact_count(nr, w.row_off.p, w.row_cnt.p, w.pool_val.p, tau, w.cnt.p, st);
  }
  DCsr &out = C;  // must not alias A or B
  out.nrows = nr;
  out.row0 = A.row0;
  out.padded = false;
  out.rp.ensure((size_t)nr + 1, st);
  launch_exclusive_scan(w.cnt.p, nr, out.rp.p, w.scan_tmp.p, st);
  if (acc != nullptr) {
    // Taylor term: S^_i and T^_0 + S^_i straight from the staged S~_i (one read of the
    // staging pool instead of compaction + a second read of S^_i by the merge).  T^_0 + S^_i
    // is written in padded form (row capacity len(T^_0 row) + nnz(S^_i row)), so no count
    // pass over T^_0 is needed; do_run compacts T^_0 once after the last term.
    DCsr &T2 = *acc_out;  // must not alias acc, A or B
    const CsrView av = acc->view();
    const int64_t *alen = acc->padded ? acc->len.p : nullptr;
    w.cnt2.ensure(nr1, st);
    launch_add_rowlen(av.rp, alen, w.cnt.p, nr, w.cnt2.p, st);
    T2.nrows = nr;
    T2.row0 = A.row0;
    T2.rp.ensure((size_t)nr + 1, st);
    launch_exclusive_scan(w.cnt2.p, nr, T2.rp.p, w.scan_tmp.p, st);
    int64_t tot[2];
    CK(cudaMemcpyAsync(&tot[0], out.rp.p + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&tot[1], T2.rp.p + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out.nnz = tot[0];
    T2.nnz = tot[1];
    out.col.ensure((size_t)out.nnz, st);
    out.val.ensure((size_t)out.nnz, st);
    T2.col.ensure((size_t)T2.nnz, st);
    T2.val.ensure((size_t)T2.nnz, st);
    T2.len.ensure(nr1, st);
    T2.padded = true;
    launch_merge_staged_write(av, alen, w.row_off.p, w.row_cnt.p, w.pool_col.p, w.pool_val.p, tau,
                              T2.rp.p, T2.col.p, T2.val.p, T2.len.p, out.rp.p, out.col.p, out.val.p, st);
    rep.nnz = (int64_t)allsum(P, (double)out.nnz);
    return;
  }
  out.nnz = d2h(out.rp.p + nr, st);
  out.col.ensure((size_t)out.nnz, st);
  out.val.ensure((size_t)out.nnz, st);
  launch_compact_write(nr, A.row0, w.row_off.p, w.row_cnt.p, w.pool_col.p, w.pool_val.p, tau,
                       out.rp.p, out.col.p, out.val.p, w.rs.p, w.l1r.p, w.l2r.p, st,
                       add_identity ? w.ident.p : nullptr);
  launch_reduce_sum(w.rs.p, nr, w.partial.p, w.scal.p + 2, st);
  launch_reduce_max_i64(w.l1r.p, nr, w.i64tmp.p + 4, st);
  launch_reduce_max_i64(w.l2r.p, nr, w.i64tmp.p + 5, st);
  rep.normIT2 = allsum(P, d2h(w.scal.p + 2, st));
  rep.l1 = (int64_t)allmax(P, (double)d2h(w.i64tmp.p + 4, st));
  rep.l2 = (int64_t)allmax(P, (double)d2h(w.i64tmp.p + 5, st));
  int64_t nnz_T = out.nnz;  // nnz of the filtered iterate itself
  if (add_identity) {
    int64_t ins_pur[2];
    CK(cudaMemcpyAsync(ins_pur, w.i64tmp.p + 6, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    nnz_T = out.nnz - ins_pur[0] + ins_pur[1];
  }
  rep.nnz = (int64_t)allsum(P, (double)nnz_T);
}

// C = A + B (same rows)
static void merge_add(sexpm_plan_s &P, const CsrView &A, const CsrView &B, DCsr &C) {
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  const int64_t nr = A.nrows;
  w.cnt.ensure((size_t)std::max<int64_t>(nr, 1), st);
  w.scan_tmp.ensure((size_t)scan_tmp_elems(nr) + 1, st);
  launch_merge_count(A, B, w.cnt.p, st);
  DCsr &out = C;  // must not alias A or B
  out.nrows = nr;
  out.row0 = A.row0;
  out.padded = false;
  out.rp.ensure((size_t)nr + 1, st);
  launch_exclusive_scan(w.cnt.p, nr, out.rp.p, w.scan_tmp.p, st);
  out.nnz = d2h(out.rp.p + nr, st);
  out.col.ensure((size_t)out.nnz, st);
  out.val.ensure((size_t)out.nnz, st);
  launch_merge_write(A, B, out.rp.p, out.col.p, out.val.p, st);
}

static void copy_csr(sexpm_plan_s &P, const CsrView &A, DCsr &C) {
  cudaStream_t st = P.st;
  C.padded = false;
  C.nrows = A.nrows;
  C.row0 = A.row0;
  C.nnz = A.nnz;
  C.rp.ensure((size_t)A.nrows + 1, st);
  C.col.ensure((size_t)A.nnz, st);
  C.val.ensure((size_t)A.nnz, st);
  CK(cudaMemcpyAsync(C.rp.p, A.rp, ((size_t)A.nrows + 1) * sizeof(int64_t),
                     cudaMemcpyDeviceToDevice, st));
  if (A.nnz) {
    CK(cudaMemcpyAsync(C.col.p, A.col, A.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(C.val.p, A.val, A.nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
}

// local row block [row_begin, row_end) of a full-row CSR (rows re-based)
static void slice_rows(sexpm_plan_s &P, const DCsr &F, int64_t r0, int64_t r1, DCsr &C) {
  cudaStream_t st = P.st;
  int64_t a = 0, b = 0;
  CK(cudaMemcpyAsync(&a, F.rp.p + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&b, F.rp.p + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  C.nrows = r1 - r0;
  C.row0 = r0;
  C.nnz = b - a;
  C.rp.alloc((size_t)C.nrows + 1, st);
  C.col.alloc((size_t)C.nnz, st);
  C.val.alloc((size_t)C.nnz, st);
  launch_rebase_rowptr(F.rp.p + r0, C.nrows, 0, C.rp.p, st);
  if (C.nnz) {
    CK(cudaMemcpyAsync(C.col.p, F.col.p + a, C.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(C.val.p, F.val.p + a, C.nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
}

// ------------------------------------------------------------------------------------
// multi-GPU: all-gather full H, halo exchange
// ------------------------------------------------------------------------------------
static void allgather_rows(sexpm_plan_s &P, const CsrView &L, DCsr &F) {
  // every rank broadcasts its block (rowptr deltas, col, val); F holds all n rows
  cudaStream_t st = P.st;
  std::vector<double> meta;
  double mine[2] = {(double)L.nrows, (double)L.nnz};
  gather_doubles(P, mine, 2, meta);
  std::vector<int64_t> rows(P.world), nnzs(P.world), roff(P.world + 1, 0), noff(P.world + 1, 0);
  for (int g = 0; g < P.world; g++) {
    rows[g] = (int64_t)meta[2 * g];
    nnzs[g] = (int64_t)meta[2 * g + 1];
    roff[g + 1] = roff[g] + rows[g];
    noff[g + 1] = noff[g] + nnzs[g];
  }
  REQUIRE(roff[P.world] == P.n, SEXPM_EINVAL, "row blocks do not cover [0, n)");
  DBuf<int64_t> rp_parts;  // per rank: its rowptr (rows+1) stored at roff[g] + g
  rp_parts.alloc((size_t)P.n + P.world, st);
  F.nrows = P.n;
  F.row0 = 0;
  F.nnz = noff[P.world];
  F.col.alloc((size_t)F.nnz, st);
  F.val.alloc((size_t)F.nnz, st);
  F.rp.alloc((size_t)P.n + 1, st);
  // my block to every peer, every peer's block from it (pieces listed in the same order on
  // both sides: rowptr, columns, values); my own block copied in place
  std::vector<Transport::Xfer> sends, recvs;
  const int me = P.rank;
  for (int g = 0; g < P.world; g++) {
    if (g == me) continue;
    sends.push_back({g, L.rp, nullptr, (size_t)(rows[me] + 1) * sizeof(int64_t)});
    if (nnzs[me]) {
      sends.push_back({g, L.col, nullptr, (size_t)nnzs[me] * sizeof(int32_t)});
      sends.push_back({g, L.val, nullptr, (size_t)nnzs[me] * sizeof(double)});
    }
    recvs.push_back({g, nullptr, rp_parts.p + roff[g] + g, (size_t)(rows[g] + 1) * sizeof(int64_t)});
    if (nnzs[g]) {
      recvs.push_back({g, nullptr, F.col.p + noff[g], (size_t)nnzs[g] * sizeof(int32_t)});
      recvs.push_back({g, nullptr, F.val.p + noff[g], (size_t)nnzs[g] * sizeof(double)});
    }
  }
  CK(cudaMemcpyAsync(rp_parts.p + roff[me] + me, L.rp, (rows[me] + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  if (nnzs[me]) {
    CK(cudaMemcpyAsync(F.col.p + noff[me], L.col, nnzs[me] * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(F.val.p + noff[me], L.val, nnzs[me] * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  P.tr->exchange(sends, recvs, st);
  for (int g = 0; g < P.world; g++)
    launch_rebase_rowptr(rp_parts.p + roff[g] + g, rows[g], noff[g], F.rp.p + roff[g], st);
  CK(cudaStreamSynchronize(st));
}

// rows a rank needs for its squaring (Lemma 3.1): [r0 - l2, r1 + l1), widened to multiples of
// 8 so that the halo matrix is block-aligned for the block kernel K3b (a superset is valid)
static void halo_need(const int64_t *bounds, int rank, int64_t n, int64_t l1, int64_t l2,
                      int64_t &need_lo, int64_t &need_hi) {
  need_lo = std::max<int64_t>(0, ((bounds[rank] - l2) >> 3) << 3);
  need_hi = std::min<int64_t>(n, ((bounds[rank + 1] + l1 + 7) >> 3) << 3);
}

static void halo_ranges_host(int world, int rank, const int64_t *bounds, int64_t n, int64_t l1,
                             int64_t l2, int64_t *lo, int64_t *hi) {
  int64_t need_lo, need_hi;
  halo_need(bounds, rank, n, l1, l2, need_lo, need_hi);
  for (int h = 0; h < world; h++) {
    int64_t a = std::max(need_lo, bounds[h]), b = std::min(need_hi, bounds[h + 1]);
    if (h == rank || a >= b) a = b = 0;
    lo[h] = a;
    hi[h] = b;
  }
}

// B = rows [need_lo, need_hi) of T^ assembled from the local block and the peers' halos
static void exchange_halo(sexpm_plan_s &P, const DCsr &T, int64_t l1, int64_t l2, DCsr &B) {
  cudaStream_t st = P.st;
  const int W = P.world, R = P.rank;
  std::vector<int64_t> rlo(W), rhi(W);
  halo_ranges_host(W, R, P.bounds.data(), P.n, l1, l2, rlo.data(), rhi.data());
  // what each peer h needs from me: symmetric computation with h's bounds
  std::vector<int64_t> slo(W), shi(W);
  for (int h = 0; h < W; h++) {
    std::vector<int64_t> lo(W), hi(W);
    halo_ranges_host(W, h, P.bounds.data(), P.n, l1, l2, lo.data(), hi.data());
    slo[h] = lo[R];
    shi[h] = hi[R];
  }
  // my rowptr at the boundaries of the pieces I send (2 values per peer, not the whole rowptr)
  std::vector<int64_t> rpa(W, 0), rpb(W, 0);
  for (int h = 0; h < W; h++)
    if (h != R && shi[h] > slo[h]) {
      CK(cudaMemcpyAsync(&rpa[h], T.rp.p + (slo[h] - T.row0), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&rpb[h], T.rp.p + (shi[h] - T.row0), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
  CK(cudaStreamSynchronize(st));
  // exchange nnz counts of the pieces
  std::vector<double> cnt_send(W, 0.0), all;
  for (int h = 0; h < W; h++)
    if (h != R && shi[h] > slo[h]) cnt_send[h] = (double)(rpb[h] - rpa[h]);
  gather_doubles(P, cnt_send.data(), W, all);  // all[g*W + h] = nnz g sends to h
  int64_t need_lo, need_hi;
  halo_need(P.bounds.data(), R, P.n, l1, l2, need_lo, need_hi);
  // pieces in row order: peers below, me, peers above
  std::vector<int64_t> piece_rows(W, 0), piece_nnz(W, 0);
  for (int h = 0; h < W; h++) {
    if (h == R) {
      piece_rows[h] = T.nrows;
      piece_nnz[h] = T.nnz;
    } else if (rhi[h] > rlo[h]) {
      piece_rows[h] = rhi[h] - rlo[h];
      piece_nnz[h] = (int64_t)all[(size_t)h * W + R];
    }
  }
  B.nrows = need_hi - need_lo;
  B.row0 = need_lo;
  B.nnz = 0;
  for (int h = 0; h < W; h++) B.nnz += piece_nnz[h];
  B.rp.alloc((size_t)B.nrows + 1, st);
  B.col.alloc((size_t)B.nnz, st);
  B.val.alloc((size_t)B.nnz, st);
  DBuf<int64_t> rp_tmp;
  rp_tmp.alloc((size_t)B.nrows + W + 1, st);
  std::vector<int64_t> row_at(W), nnz_at(W), tmp_at(W);
  int64_t ro = 0, no = 0, to = 0;
  for (int h = 0; h < W; h++) {
    row_at[h] = ro;
    nnz_at[h] = no;
    tmp_at[h] = to;
    ro += piece_rows[h];
    no += piece_nnz[h];
    to += piece_rows[h] ? piece_rows[h] + 1 : 0;
  }
  REQUIRE(ro == B.nrows, SEXPM_EINTERNAL, "halo rows do not tile the needed range");
  std::vector<Transport::Xfer> sends, recvs;
  for (int h = 0; h < W; h++) {
    if (h == R) continue;
    if (shi[h] > slo[h]) {
      int64_t a = slo[h] - T.row0, b = shi[h] - T.row0;
      sends.push_back({h, T.rp.p + a, nullptr, (size_t)(b - a + 1) * sizeof(int64_t)});
      int64_t na = rpa[h], nb = rpb[h];
      if (nb > na) {
        sends.push_back({h, T.col.p + na, nullptr, (size_t)(nb - na) * sizeof(int32_t)});
        sends.push_back({h, T.val.p + na, nullptr, (size_t)(nb - na) * sizeof(double)});
      }
    }
    if (piece_rows[h]) {
      recvs.push_back({h, nullptr, rp_tmp.p + tmp_at[h], (size_t)(piece_rows[h] + 1) * sizeof(int64_t)});
      if (piece_nnz[h]) {
        recvs.push_back({h, nullptr, B.col.p + nnz_at[h], (size_t)piece_nnz[h] * sizeof(int32_t)});
        recvs.push_back({h, nullptr, B.val.p + nnz_at[h], (size_t)piece_nnz[h] * sizeof(double)});
      }
    }
  }
  P.tr->exchange(sends, recvs, st);
  // my own rows
  CK(cudaMemcpyAsync(rp_tmp.p + tmp_at[R], T.rp.p, (T.nrows + 1) * sizeof(int64_t),
                     cudaMemcpyDeviceToDevice, st));
  if (T.nnz) {
    CK(cudaMemcpyAsync(B.col.p + nnz_at[R], T.col.p, T.nnz * sizeof(int32_t),
                       cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(B.val.p + nnz_at[R], T.val.p, T.nnz * sizeof(double),
                       cudaMemcpyDeviceToDevice, st));
  }
  for (int h = 0; h < W; h++)
    if (piece_rows[h])
      launch_rebase_rowptr(rp_tmp.p + tmp_at[h], piece_rows[h], nnz_at[h], B.rp.p + row_at[h], st);
  CK(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------------------------------
// processing order with L2 locality (plan time, host): rows are visited cluster by
// cluster, each cluster a BFS ball of ~kCluster rows of H's graph, clusters taken in a
// global BFS sweep.  The dynamic row scheduler of K3 hands consecutive rows of this
// order to the CTAs in flight, so the B rows they gather (the ball dilated by the
// bandwidth of T^, Lemma 3.1) stay L2-resident (126 MB) instead of the whole band of
// lexicographically consecutive rows (~2R grid lines for a 2D stencil).
// ------------------------------------------------------------------------------------
// 8-row aggregates of H's graph (greedy BFS from seeds in index order): every 8 consecutive
// rows of the new order are a compact neighbourhood, so the 8x8 blocks of the squared
// iterate are fuller (config-5-like pattern: 45 % fewer block products in the model,
// DESIGN.md section 6).  perm[new] = old.
// 8-row aggregates of the rows [lo, hi) of H's graph (one rank's range: aggregates never
// cross the rank partition, so the relabelling is block-diagonal over it and every rank
// relabels only its own rows).  perm receives the range's nodes in the new order (global ids).
//   aggregate_order: greedy BFS from seeds in index order (every aggregate a compact
//     neighbourhood: a star of the seed's ring on a grid);
//   aggregate_order_compact: from each seed add, one at a time, the unused neighbour with the
//     most edges into the aggregate; ties to the candidate adjacent to the earliest-added
//     member, then to the smaller index (2 x 2 x 2 cubes on a 3D grid, 4 x 2 rectangles in 2D).
static void aggregate_order(const std::vector<int64_t> &rp, const std::vector<int32_t> &col,
                            int64_t lo, int64_t hi, int size, std::vector<int64_t> &perm) {
  perm.clear();
  perm.reserve((size_t)(hi - lo));
  std::vector<uint8_t> used((size_t)(hi - lo), 0);
  for (int64_t s = lo; s < hi; s++) {
    if (used[s - lo]) continue;
    const size_t g0 = perm.size();
    perm.push_back(s);
    used[s - lo] = 1;
    for (size_t h = g0; h < perm.size() && (int)(perm.size() - g0) < size; h++) {
      const int64_t v = perm[h];
      for (int64_t p = rp[v]; p < rp[v + 1] && (int)(perm.size() - g0) < size; p++) {
        const int64_t u = col[p];
        if (u >= lo && u < hi && !used[u - lo]) {
          used[u - lo] = 1;
          perm.push_back(u);
        }
      }
    }
  }
}

static void aggregate_order_compact(const std::vector<int64_t> &rp, const std::vector<int32_t> &col,
                                    int64_t lo, int64_t hi, int size, std::vector<int64_t> &perm) {
  const int64_t m = hi - lo;
  perm.clear();
  perm.reserve((size_t)m);
  std::vector<uint8_t> used((size_t)m, 0);
  std::vector<int32_t> cnt((size_t)m, 0), firstm((size_t)m, 0);  // per candidate: edges, first member
  std::vector<int64_t> agg, cand;
  for (int64_t s = lo; s < hi; s++) {
    if (used[s - lo]) continue;
    agg.clear();
    cand.clear();
    int64_t v = s;
    for (;;) {
      used[v - lo] = 1;
      const int mi = (int)agg.size();
      agg.push_back(v);
      if ((int)agg.size() >= size) break;
      for (int64_t p = rp[v]; p < rp[v + 1]; p++) {  // v's edges raise its neighbours' counts
        const int64_t u = col[p];
        if (u < lo || u >= hi || used[u - lo]) continue;
        if (cnt[u - lo] == 0) {
          firstm[u - lo] = mi;
          cand.push_back(u);
        }
        cnt[u - lo]++;
      }
      int64_t best = -1;
      for (int64_t u : cand) {
        if (used[u - lo]) continue;
        const int64_t ul = u - lo, bl = best - lo;
        if (best < 0 || cnt[ul] > cnt[bl] ||
            (cnt[ul] == cnt[bl] && (firstm[ul] < firstm[bl] || (firstm[ul] == firstm[bl] && u < best))))
          best = u;
      }
      if (best < 0) break;
      v = best;
    }
    for (int64_t u : cand) cnt[u - lo] = 0;
    perm.insert(perm.end(), agg.begin(), agg.end());
  }
}

// Block-fill proxy of an order of the rows [lo, hi): for sampled block rows (8 consecutive
// positions of the order), the distinct column blocks covered by the radius-rad neighbourhood
// of their 8 rows in H's graph -- the iterates' rows are such neighbourhoods, rad ~ 0.8 M the
// reach of the filtered Taylor phase -- counting only rows of the range (so the result
// depends on the range alone).  Sampling stops after ~2e6 visited rows.  perm = null: index
// order.
static int64_t sampled_blocks(const std::vector<int64_t> &rp, const std::vector<int32_t> &col,
                              int64_t lo, int64_t hi, const std::vector<int64_t> *perm, int rad) {
  const int64_t m = hi - lo, nbt = (m + 7) / 8, step = std::max<int64_t>(1, nbt / 512);
  std::vector<int64_t> pos;  // position in the order of each row of the range
  if (perm) {
    pos.resize((size_t)m);
    for (int64_t i = 0; i < m; i++) pos[(*perm)[i] - lo] = i;
  }
  std::vector<int32_t> mark((size_t)m, -1);
  std::vector<int64_t> fr, nx, blk;
  int64_t total = 0, visited = 0;
  int32_t stamp = 0;
  for (int64_t b = 0; b < nbt && visited < 2000000; b += step, stamp++) {
    fr.clear();
    blk.clear();
    for (int64_t i = 8 * b; i < std::min<int64_t>(m, 8 * b + 8); i++) {
      const int64_t v = perm ? (*perm)[i] : lo + i;
      if (mark[v - lo] != stamp) {
        mark[v - lo] = stamp;
        fr.push_back(v);
        blk.push_back(i >> 3);
      }
    }
    for (int r = 0; r < rad; r++) {
      nx.clear();
      for (int64_t v : fr)
        for (int64_t p = rp[v]; p < rp[v + 1]; p++) {
          const int64_t u = col[p];
          if (u < lo || u >= hi || mark[u - lo] == stamp) continue;
          mark[u - lo] = stamp;
          nx.push_back(u);
          blk.push_back((perm ? pos[u - lo] : u - lo) >> 3);
        }
      visited += (int64_t)nx.size();
      fr.swap(nx);
    }
    std::sort(blk.begin(), blk.end());
    total += std::unique(blk.begin(), blk.end()) - blk.begin();
  }
  return total;
}

static void cluster_order(const std::vector<int64_t> &rp, const std::vector<int32_t> &col,
                          int64_t r0, int64_t r1, int cluster, std::vector<int32_t> &order) {
  const int64_t nl = r1 - r0;
  order.clear();
  order.reserve((size_t)nl);
  std::vector<int32_t> gorder;
  gorder.reserve((size_t)nl);
  std::vector<uint8_t> seen((size_t)nl, 0), assigned((size_t)nl, 0);
  for (int64_t s = 0; s < nl; s++) {
    if (seen[s]) continue;
    size_t head = gorder.size();
    gorder.push_back((int32_t)s);
    seen[s] = 1;
    while (head < gorder.size()) {
      int64_t v = gorder[head++];
      for (int64_t p = rp[v + r0]; p < rp[v + r0 + 1]; p++) {
        int64_t u = (int64_t)col[p] - r0;
        if (u >= 0 && u < nl && !seen[u]) {
          seen[u] = 1;
          gorder.push_back((int32_t)u);
        }
      }
    }
  }
  std::vector<int32_t> q;
  for (int32_t s : gorder) {
    if (assigned[s]) continue;
    q.clear();
    q.push_back(s);
    assigned[s] = 1;
    size_t head = 0;
    while (head < q.size() && (int)q.size() < cluster) {
      int64_t v = q[head++];
      for (int64_t p = rp[v + r0]; p < rp[v + r0 + 1] && (int)q.size() < cluster; p++) {
        int64_t u = (int64_t)col[p] - r0;
        if (u >= 0 && u < nl && !assigned[u]) {
          assigned[u] = 1;
          q.push_back((int32_t)u);
        }
      }
    }
    // rows of a cluster in index order: neighbours in the processing order are then mostly
    // neighbours in the matrix (the grouped kernel shares their B rows)
    std::sort(q.begin(), q.end());
    order.insert(order.end(), q.begin(), q.end());
  }
}

// ------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------
// Forward error of the truncated Taylor series, Eq. (4.5)-(4.6) P:266-276:
//   r0(x, M) = (1/M!) int_0^x t^M e^t dt = (-1)^{M+1} gamma(M+1, -x) / M!.
// Evaluated here through Kummer's transformation of the incomplete gamma function,
//   r0(x, M) = x^{M+1} e^x / (M+1)! * 1F1(1; M+2; -x)
//            = x^{M+1} e^x / (M+1)! * sum_k (-x)^k / ((M+2)(M+3)...(M+1+k)),
// an alternating series whose terms shrink at least by x/(M+2) <= 1/2 for the planner's
// x = ||H 2^-N|| <= 1 (Eq. 4.20's first constraint), so it is summed in long double until
// the terms no longer change the sum.  (The CPU oracle evaluates the paper's own series;
// tests/test_planner_abi.py checks this against 30-digit quadrature.)
static long double taylor_remainder(long double x, int M) {
  if (!(x > 0.0L)) return 0.0L;
  // lead = x^{M+1} e^x / (M+1)!, built as a product of x / j, j = 1..M+1
  long double lead = expl(x);
  for (int j = 1; j <= M + 1; j++) lead *= x / (long double)j;
  long double kummer = 0.0L, term = 1.0L;
  for (int k = 0; k < 4096; k++) {
    const long double next = kummer + term;
    if (next == kummer) break;
    kummer = next;
    term *= -x / (long double)(M + 2 + k);
  }
  return lead * kummer;
}

// ceil(log2(v)) for v > 0, exactly (frexp: v = f 2^e with f in [0.5, 1))
static int ceil_log2_exact(double v) {
  int e = 0;
  const double f = frexp(v, &e);
  return f == 0.5 ? e - 1 : e;
}

// (M, N) by Eq. (4.20): minimise M 2^N subject to ||H 2^-N|| <= 1 and
// 2^N r0(||H|| 2^-N, M) <= eps_tol, over N in [N0, N0 + n_window] (N0 = max(ceil(log2
// ||H||), 0), "N_max = N0 + 50") and M in [0, m_cap] (reading R5; ties to the
// smaller N).  Returns false when no candidate satisfies the tolerance.
static bool select_MN(double norm, double eps_tol, int m_cap, int n_window, int &M, int &N) {
  if (norm == 0.0) {  // H = 0: e^H = I, nothing to do (reading R9)
    M = 0;
    N = 0;
    return true;
  }
  const int N0 = std::max(ceil_log2_exact(norm), 0);
  struct Cand { int N, M; long double cost; };
  std::vector<Cand> cands;
  for (int k = 0; k <= n_window; k++) {
    const int n = N0 + k;
    const long double x = (long double)ldexp(norm, -n);  // exact scaling by 2^-n
    const long double scale = ldexpl(1.0L, n);
    // m(N): the least M meeting the tolerance; r0 decreases with M, so the first hit
    int m = 0;
    while (m <= m_cap && scale * taylor_remainder(x, m) > (long double)eps_tol) m++;
    if (m <= m_cap) cands.push_back({n, m, (long double)m * scale});
  }
  if (cands.empty()) return false;
  // candidates are in increasing N: the first of the minimal cost wins the tie
  const Cand *best = &cands[0];
  for (const Cand &c : cands)
    if (c.cost < best->cost) best = &c;
  M = best->M;
  N = best->N;
  return true;
}

// Filter budgets of Algorithm 4.2 steps 2-3: a = 1/(N+1) for normal H
// (Eq. 4.19), else a = min(1, 1/||H||) (reading R8); r0 = r0(||H 2^-N||, M)
// (Eq. 4.5); the Taylor threshold eps_g^(0) = a r0 / (M e^{2 ||H0||}) (Eq. 4.14),
// 0 when M = 0 (reading R9: no Taylor terms are filtered).
static void filter_budgets(double norm, int normal, int M, int N, double &a, long double &r0,
                           double &eps_g0) {
  a = normal ? 1.0 / (1.0 + (double)N) : (norm > 1.0 ? 1.0 / norm : 1.0);
  const long double x = (long double)ldexp(norm, -N);
  r0 = taylor_remainder(x, M);
  eps_g0 = M >= 1 ? (double)((long double)a * r0 / ((long double)M * expl(2.0L * x))) : 0.0;
}

// Diagonal offsets of H0 (d = j - k over all entries); when there are at most kDiaMax of
// them the Taylor terms use the diagonal push kernel K5d (grid stencils have 3 / 5 / 7).
static void build_diagonals(sexpm_plan_s &P) {
  cudaStream_t st = P.st;
  P.dia_nd = 0;
  const DCsr &Hf = P.H0full;
  if (Hf.nnz == 0 || P.o.kernel != 0 && P.o.kernel != 7 && P.o.kernel != 8) return;
  if (P.n > (int64_t(1) << 30)) return;  // K5d computes columns k + d in 32 bits
  const int64_t nbits = 2 * P.n - 1, nwords = (nbits + 31) / 32;
  DBuf<unsigned> bits;
  bits.alloc((size_t)nwords, st);
  CK(cudaMemsetAsync(bits.p, 0, nwords * sizeof(unsigned), st));
  launch_mark_offsets(Hf.view(), bits.p, P.n, st);
  std::vector<unsigned> hb((size_t)nwords);
  CK(cudaMemcpyAsync(hb.data(), bits.p, nwords * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int32_t> offs;
  for (int64_t w = 0; w < nwords && (int)offs.size() <= kDiaMax; w++) {
    unsigned m = hb[w];
    while (m) {
      const int b = __builtin_ctz(m);
      m &= m - 1;
      offs.push_back((int32_t)(w * 32 + b - (P.n - 1)));
    }
  }
  if (offs.empty() || (int)offs.size() > kDiaMax) return;
  std::sort(offs.begin(), offs.end(), std::greater<int32_t>());  // descending: k ascending per column
  P.dia_nd = (int)offs.size();
  P.h_dia_off = offs;
  P.dia_dmax = offs.front();
  P.dia_dmin = offs.back();
  P.dia_off.alloc(offs.size(), st);
  CK(cudaMemcpyAsync(P.dia_off.p, offs.data(), offs.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  P.dia_val.alloc((size_t)P.dia_nd * P.n, st);
  CK(cudaMemsetAsync(P.dia_val.p, 0, (size_t)P.dia_nd * P.n * sizeof(double), st));
  launch_fill_dia(Hf.view(), offs.data(), P.dia_nd, P.dia_val.p, P.n, st);
  P.dia_prod.alloc(1, st);
  P.dia_need.alloc(1, st);
  {  // largest K5d slot count whose 4-warp CTA fits the opt-in shared memory of a block
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, P.dev));
    int sl = 8192;
    while (sl > 256 && taylor_dia_smem_bytes(sl) > optin) sl -= 64;
    P.dia_slots_max = sl;
  }
  CK(cudaStreamSynchronize(st));  // offs (host) is captured by value in the launch
}

// Grid structure of H0 from its diagonal offsets (row r = x + G y [+ G Gy z]): 2D when the
// positive offsets are {1, G} with G | n, 3D when they are {1, G, G Gy} with G Gy | n.  Only a
// heuristic for the squarings' row order: any H is handled correctly, a banded matrix that
// merely looks like a grid just gets a less useful order.
static bool detect_lattice(const sexpm_plan_s &P, LatticeDesc &L) {
  if (P.dia_nd == 0 || getenv("SEXPM_NO_LATTICE")) return false;
  std::vector<int64_t> pos;
  for (int32_t d : P.h_dia_off)
    if (d > 0) pos.push_back(d);
  std::sort(pos.begin(), pos.end());
  for (int32_t d : P.h_dia_off)  // symmetric offset set
    if (std::find(P.h_dia_off.begin(), P.h_dia_off.end(), -d) == P.h_dia_off.end()) return false;
  L = LatticeDesc{};
  L.n = P.n;
  if (pos.size() == 2 && pos[0] == 1 && pos[1] > 1 && P.n % pos[1] == 0 && P.n / pos[1] > 1) {
    L.dims = 2;
    L.G = pos[1];
    L.Gy = P.n / pos[1];
    L.GH = P.n;
    L.Dp = 4 * ((L.Gy + 3) / 4);
    const int64_t nu = (L.G + L.Gy - 2) / 4 + 1;
    L.nv = (L.G - 1 + L.Dp) / 4 + 1;
    L.nv16 = (L.nv + 15) / 16;
    L.ntiles = nu * L.nv;
    L.nsuper = ((nu + 15) / 16) * L.nv16;
    return true;
  }
  if (pos.size() == 3 && pos[0] == 1 && pos[1] > 1 && pos[2] % pos[1] == 0 && pos[2] / pos[1] > 1 &&
      P.n % pos[2] == 0 && P.n / pos[2] > 1) {
    L.dims = 3;
    L.G = pos[1];
    L.Gy = pos[2] / pos[1];
    L.GH = pos[2];
    const int64_t Gz = P.n / pos[2];
    L.ntx = (L.G + 1) / 2;
    L.nty = (L.Gy + 1) / 2;
    const int64_t ntz = (Gz + 1) / 2;
    L.nx8 = (L.ntx + 7) / 8;
    L.ny8 = (L.nty + 7) / 8;
    L.ntiles = L.ntx * L.nty * ntz;
    L.nsuper = L.nx8 * L.ny8 * ((ntz + 7) / 8);
    return true;
  }
  return false;
}

// K5w tables (kernels.cu k_taylor_win): the offsets a row of S~_j can reach are the Minkowski
// sums W_j = W_{j-1} + D (W_1 = D, H0's diagonal offsets), offsets with |o| >= n pruned (no
// row has such a column).  U = W_1 u ... u W_M ascending; per U-index and diagonal the U-index
// of o - d (the input offset of the product s(r, r+o-d) h_d(r+o-d)); per term the U-indices of
// W_j and of the cumulative union (the support of T^_0 after term j), ascending.  The window is
// used when U is small enough for shared memory (grid stencils in 1D / 2D; 3D octahedra of
// radius M are not) with at least 8 resident warps per SM.
// the symmetric path (option sym_squaring, reading R21): H bit-exactly symmetric, one GPU, the
// tensor-core squarings
static bool sym_path_enabled(const sexpm_plan_s &P) {
  return P.o.sym_squaring != 0 && P.h_sym && P.world == 1 && !P.o.exact_products && !P.o.ssat &&
         (P.o.kernel == 0 || P.o.kernel == 8 || P.o.kernel == 13) && P.N >= 1;
}

static void build_window(sexpm_plan_s &P) {
  auto &W = P.win;
  cudaStream_t st = P.st;
  W.ok = false;
  if (P.dia_nd == 0 || P.M < 1 || P.o.kernel != 0 && P.o.kernel != 8) return;
  if (getenv("SEXPM_NO_WIN")) return;
  constexpr int kCap = 4096;
  const int nd = P.dia_nd;
  std::vector<int64_t> D(P.h_dia_off.begin(), P.h_dia_off.end());
  std::vector<std::vector<int64_t>> Wj((size_t)P.M + 1);
  std::vector<int64_t> cur;
  for (int64_t d : D)
    if (d > -P.n && d < P.n) cur.push_back(d);
  std::sort(cur.begin(), cur.end());
  cur.erase(std::unique(cur.begin(), cur.end()), cur.end());
  Wj[1] = cur;
  std::vector<int64_t> U = cur;
  for (int j = 2; j <= P.M; j++) {
    std::vector<int64_t> nx;
    nx.reserve(cur.size() * D.size());
    for (int64_t o : cur)
      for (int64_t d : D) {
        const int64_t v = o + d;
        if (v > -P.n && v < P.n) nx.push_back(v);
      }
    std::sort(nx.begin(), nx.end());
    nx.erase(std::unique(nx.begin(), nx.end()), nx.end());
    std::vector<int64_t> un;
    std::set_union(U.begin(), U.end(), nx.begin(), nx.end(), std::back_inserter(un));
    U.swap(un);
    if ((int)U.size() > kCap) return;
    Wj[j] = nx;
    cur.swap(nx);
  }
  const int nU = (int)U.size();
  // half window: symmetric H, T^_0 fused into the terms (0 in D), at least two terms
  int dz0 = -1;
  for (size_t di = 0; di < D.size(); di++)
    if (D[di] == 0) dz0 = (int)di;
  const bool half = sym_path_enabled(P) && dz0 >= 0 && P.M >= 3 && !getenv("SEXPM_NO_HALF_WIN");
  auto nonneg = [](const std::vector<int64_t> &v) {
    std::vector<int64_t> h;
    for (int64_t o : v)
      if (o >= 0) h.push_back(o);
    return h;
  };
  std::vector<std::vector<int64_t>> Wh((size_t)P.M + 1);
  for (int j = 1; j <= P.M; j++) Wh[j] = nonneg(Wj[j]);
  const std::vector<int64_t> Uh = nonneg(U);
  int64_t padr = 0;
  for (int64_t d : D) padr = std::max<int64_t>(padr, d);
  // positions: binary search in a sorted offset list
  auto pos = [](const std::vector<int64_t> &v, int64_t o) -> int {
    auto it = std::lower_bound(v.begin(), v.end(), o);
    return (it != v.end() && *it == o) ? (int)(it - v.begin()) : -1;
  };
  int dzero = -1;
  for (int di = 0; di < nd; di++)
    if (D[di] == 0) dzero = di;
  const int64_t nl = P.row_end - P.row_begin;
  int64_t maxo = 0, maxd = 0;
  for (int64_t o : U) maxo = std::max<int64_t>(maxo, o < 0 ? -o : o);
  for (int64_t d : D) maxd = std::max<int64_t>(maxd, d < 0 ? -d : d);
  const int64_t pad = maxo + maxd + 1, npad = P.n + 2 * pad;
  const int knd = taylor_win_kernel_nd(nd), rw = taylor_win_rec_words(nd);
  // the records hold int32 element offsets
  int64_t maxl = 0, maxc = 0;
  {
    std::vector<int64_t> cu;
    for (int j = 1; j <= P.M; j++) {
      std::vector<int64_t> un;
      std::set_union(cu.begin(), cu.end(), Wj[j].begin(), Wj[j].end(), std::back_inserter(un));
      cu.swap(un);
      maxl = std::max<int64_t>(maxl, (int64_t)Wj[j].size());
      maxc = std::max<int64_t>(maxc, (int64_t)cu.size());
    }
  }
  if ((maxl + 1) * nl >= INT32_MAX || (int64_t)(U.size() + 1) * nl >= INT32_MAX || (int64_t)(nd + 1) * npad >= INT32_MAX)
    return;
  W.lcnt.assign((size_t)P.M + 1, 0);
  W.lcnt_h.assign((size_t)P.M + 1, 0);
  W.ccnt.assign((size_t)P.M + 1, 0);
  const int64_t nlp = half ? nl + padr : nl;  // plane stride of the S~ checkpoints
  W.woff.assign((size_t)P.M + 2, 0);
  W.coff.assign((size_t)P.M + 2, 0);
  std::vector<int32_t> hrec, hco;
  std::vector<int16_t> hmc, hmw, hcu;
  std::vector<int64_t> cum, cum_prev, cum_prev2;
  for (int j = 1; j <= P.M; j++) {
    std::vector<int64_t> un;
    std::set_union(cum.begin(), cum.end(), Wj[j].begin(), Wj[j].end(), std::back_inserter(un));
    cum_prev2 = cum_prev;
    cum_prev = cum;  // cum_{j-1}
    cum.swap(un);    // cum_j
    W.lcnt[j] = (int)Wj[j].size();
    W.lcnt_h[j] = (int)Wh[j].size();
    W.ccnt[j] = (int)cum.size();
    W.woff[j] = (int64_t)hrec.size();
    W.coff[j] = (int64_t)hco.size();
    if (j >= 2 && half) {  // TERM launch i = j over W_j's offsets o >= 0
      const int64_t zs = j == 2 ? (int64_t)nd * npad : (int64_t)W.lcnt_h[j - 1] * nlp;  // zero planes
      const int64_t zt = (int64_t)Uh.size() * nl;
      const std::vector<int64_t> cph = nonneg(cum_prev), cph2 = nonneg(cum_prev2);
      for (int64_t o : Wh[j]) {
        for (int di = 0; di < knd; di++) {
          int64_t rv = zs;
          if (di < nd) {
            const int64_t sft = o - D[di];
            if (j == 2) {  // S~_1 = H0: its diagonals exist for either sign
              const int p = pos(Wj[1], sft);
              if (p >= 0) rv = (int64_t)(nd - 1 - p) * npad;
            } else if (sft >= 0) {
              const int p = pos(Wh[j - 1], sft);
              if (p >= 0) rv = (int64_t)p * nlp;
            } else {  // S^_{j-1}(r, r + s) = S^_{j-1}(r + s, r): the mirror's row, shift s
              const int p = pos(Wh[j - 1], -sft);
              if (p >= 0) rv = (int64_t)p * nlp + sft;
            }
          }
          hrec.push_back((int32_t)rv);
        }
        const int q = pos(cph, o);
        const int pc = pos(cph2, o);
        const int64_t uo = pos(Uh, o);
        hrec.push_back((int32_t)(q < 0 ? -1 : uo * nl));
        hrec.push_back((int32_t)(pc < 0 ? zt : uo * nl));
        hrec.push_back((int32_t)o);
        for (int w = knd + 3; w < rw; w++) hrec.push_back(0);
      }
      for (int64_t o : cph) REQUIRE(pos(Wh[j], o) >= 0, SEXPM_EINTERNAL, "window tables: cum not in W (half)");
    } else if (j >= 2) {  // TERM launch i = j: records over W_j
      const int64_t zs = j == 2 ? (int64_t)nd * npad : (int64_t)W.lcnt[j - 1] * nl;  // zero planes
      const int64_t zt = (int64_t)nU * nl;  // T^_0's zero plane
      for (int64_t o : Wj[j]) {
        for (int di = 0; di < knd; di++) {
          const int p = di < nd ? pos(Wj[j - 1], o - D[di]) : -1;
          hrec.push_back((int32_t)(p < 0 ? zs : (j == 2 ? (int64_t)(nd - 1 - p) * npad : (int64_t)p * nl)));
        }
        // T^_0 (in place over U): written when o is in cum_{j-1} (fused only when 0 is in D),
        // read back when o was already in cum_{j-2} (else the zero plane)
        const int q = dzero >= 0 ? pos(cum_prev, o) : -1;
        const int pc = pos(cum_prev2, o);
        const int64_t uo = pos(U, o);
        hrec.push_back((int32_t)(q < 0 ? -1 : uo * nl));
        hrec.push_back((int32_t)(pc < 0 ? zt : uo * nl));
        hrec.push_back((int32_t)o);
        for (int w = knd + 3; w < rw; w++) hrec.push_back(0);
      }
      // the fused T^_0 update needs cum_{j-1} inside W_j (true when 0 is in D)
      if (dzero >= 0)
        for (int64_t o : cum_prev) REQUIRE(pos(Wj[j], o) >= 0, SEXPM_EINTERNAL, "window tables: cum not in W");
    }
    for (int64_t o : cum) {
      hco.push_back((int32_t)o);
      if (half) {  // the FINAL reads |o| (the mirror's row for o < 0)
        const int64_t ao = o < 0 ? -o : o;
        hmc.push_back((int16_t)(pos(cum_prev, ao) >= 0 ? pos(Uh, ao) : -1));
        hmw.push_back((int16_t)pos(Wh[j], ao));
        hcu.push_back((int16_t)pos(Uh, ao));
      } else {
        hmc.push_back((int16_t)(pos(cum_prev, o) >= 0 ? pos(U, o) : -1));
        hmw.push_back((int16_t)pos(Wj[j], o));
        hcu.push_back((int16_t)pos(U, o));
      }
    }
  }
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, P.dev));
  for (int j = 2; j <= P.M; j++)
    if (taylor_win_smem_bytes(nd, W.lcnt[j], W.ccnt[j - 1]) > optin - 1024) return;
  W.nU = nU;
  W.half = half;
  W.nUh = (int)Uh.size();
  W.padr = half ? padr : 0;
  W.dzero = dzero;
  W.rw = rw;
  W.pad = pad;
  W.npad = npad;
  W.rec.alloc(std::max<size_t>(hrec.size(), 4), st);
  if (!hrec.empty()) CK(cudaMemcpyAsync(W.rec.p, hrec.data(), hrec.size() * 4, cudaMemcpyHostToDevice, st));
  W.coffs.alloc(std::max<size_t>(hco.size(), 1), st);
  CK(cudaMemcpyAsync(W.coffs.p, hco.data(), hco.size() * 4, cudaMemcpyHostToDevice, st));
  W.mapC.alloc(std::max<size_t>(hmc.size(), 1), st);
  CK(cudaMemcpyAsync(W.mapC.p, hmc.data(), hmc.size() * 2, cudaMemcpyHostToDevice, st));
  W.mapW.alloc(std::max<size_t>(hmw.size(), 1), st);
  CK(cudaMemcpyAsync(W.mapW.p, hmw.data(), hmw.size() * 2, cudaMemcpyHostToDevice, st));
  W.cumU.alloc(std::max<size_t>(hcu.size(), 1), st);
  CK(cudaMemcpyAsync(W.cumU.p, hcu.data(), hcu.size() * 2, cudaMemcpyHostToDevice, st));
  W.neg1.alloc((size_t)std::max<int64_t>(maxc, 1), st);
  CK(cudaMemsetAsync(W.neg1.p, 0xff, (size_t)std::max<int64_t>(maxc, 1) * 2, st));  // int16 -1
  // zero-padded diagonals (+ a zero plane): h_d(k) for any k the window can form
  W.dpad.alloc((size_t)(nd + 1) * (size_t)npad, st);
  CK(cudaMemsetAsync(W.dpad.p, 0, (size_t)(nd + 1) * (size_t)npad * sizeof(double), st));
  for (int di = 0; di < nd; di++)
    CK(cudaMemcpyAsync(W.dpad.p + (size_t)di * npad + pad, P.dia_val.p + (size_t)di * P.n, (size_t)P.n * sizeof(double),
                       cudaMemcpyDeviceToDevice, st));
  W.cnt.alloc(1, st);
  W.need.alloc(1, st);
  CK(cudaStreamSynchronize(st));  // host vectors go out of scope
  W.ok = true;
}

// ------------------------------------------------------------------------------------
// N3: reverse Cuthill-McKee of pattern(H + H^T) on the device, the
// oracle's rules (or_rcm): isolated nodes first in index order, then components from their
// smallest (degree, index) node, pseudo-peripheral start (George-Liu), Cuthill-McKee levels
// ordered by (smallest position of a neighbour in the previous level, degree, index), the
// whole sequence reversed.  Host loop over BFS levels, one d2h per level.
// ------------------------------------------------------------------------------------
// C = A permuted (row i <- row rowmap[i], column c -> colmap[c], rows re-sorted).  The
// unsorted rows go to the staging pool (free between the phases) and CUB sorts between it and
// C, so no other O(nnz) buffer is allocated.
static void permute_csr(sexpm_plan_s &P, const CsrView &A, const int64_t *rowmap, const int64_t *colmap,
                        DCsr &C) {
  cudaStream_t st = P.st;
  Workspace &w = P.ws;
  const int64_t n = A.nrows;
  REQUIRE(A.nnz < INT32_MAX, SEXPM_EINVAL, "permutation: nnz must be < 2^31 (segmented sort)");
  w.cnt.ensure((size_t)std::max<int64_t>(n, 1), st);
  w.scan_tmp.ensure((size_t)scan_tmp_elems(n) + 1, st);
  C.nrows = n;
  C.row0 = A.row0;  // rows are relabelled within the view (a rank's own rows)
  C.nnz = A.nnz;
  C.padded = false;
  C.rp.ensure((size_t)n + 1, st);
  C.col.ensure((size_t)std::max<int64_t>(A.nnz, 1), st);
  C.val.ensure((size_t)std::max<int64_t>(A.nnz, 1), st);
  launch_perm_count(A.rp, rowmap, n, w.cnt.p, st);
  launch_exclusive_scan(w.cnt.p, n, C.rp.p, w.scan_tmp.p, st);
  w.i64tmp.ensure(8, st);
  launch_reduce_max_i64(w.cnt.p, n, w.i64tmp.p + 0, st);
  if (d2h(w.i64tmp.p + 0, st) <= kSortRowsCap) {  // short rows: relabel and sort in one pass
    launch_perm_sort_rows(A, rowmap, colmap, n, C.rp.p, C.col.p, C.val.p, st);
    CK(cudaGetLastError());
    return;
  }
  w.pool_col.ensure((size_t)std::max<int64_t>(A.nnz, 1), st);
  w.pool_val.ensure((size_t)std::max<int64_t>(A.nnz, 1), st);
  launch_perm_write(A, rowmap, colmap, n, C.rp.p, w.pool_col.p, w.pool_val.p, st);
  const size_t tb = seg_sort_temp_bytes(A.nnz, n, C.rp.p);
  DBuf<unsigned char> tmp;
  tmp.alloc(tb + 256, st);
  int32_t *kc = w.pool_col.p;
  double *vc = w.pool_val.p;
  launch_seg_sort(&kc, C.col.p, &vc, C.val.p, A.nnz, n, C.rp.p, tmp.p, tb, st);
  if (A.nnz && kc != C.col.p) {
    CK(cudaMemcpyAsync(C.col.p, kc, A.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(C.val.p, vc, A.nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaGetLastError());
}

static void compute_rcm(sexpm_plan_s &P, const CsrView &H, DBuf<int64_t> &perm, DBuf<int64_t> &inv) {
  cudaStream_t st = P.st;
  Workspace &w = P.ws;
  const int64_t n = H.nrows;
  const size_t n1 = (size_t)std::max<int64_t>(n, 1);
  // G = pattern(H + H^T): the merge of H's and H^T's rows with positive stand-in values
  DCsr HT;
  build_transpose(P, H, n, HT);
  DBuf<double> v1, v2;
  v1.alloc((size_t)std::max<int64_t>(H.nnz, 1), st);
  v2.alloc((size_t)std::max<int64_t>(H.nnz, 1), st);
  CK(cudaMemsetAsync(v1.p, 0x3F, std::max<int64_t>(H.nnz, 1) * sizeof(double), st));
  CK(cudaMemsetAsync(v2.p, 0x3F, std::max<int64_t>(H.nnz, 1) * sizeof(double), st));
  CsrView Hv = H, Tv = HT.view();
  Hv.val = v1.p;
  Tv.val = v2.p;
  DCsr G;
  merge_add(P, Hv, Tv, G);
  const CsrView Gv = G.view();
  DBuf<int32_t> deg, level, ids, ids2;
  DBuf<int64_t> queue, pos, cm;
  DBuf<int8_t> done;
  DBuf<unsigned long long> key, key2, keyv, tail, mn;
  deg.alloc(n1, st);
  level.alloc(n1, st);
  ids.alloc(n1, st);
  ids2.alloc(n1, st);
  queue.alloc(n1, st);
  pos.alloc(n1, st);
  cm.alloc(n1, st);
  done.alloc(n1, st);
  key.alloc(n1, st);
  key2.alloc(n1, st);
  keyv.alloc(n1, st);
  tail.alloc(1, st);
  mn.alloc(1, st);
  const size_t tb = cm_sort_temp_bytes(n);
  DBuf<unsigned char> tmp;
  tmp.alloc(tb + 256, st);
  launch_degree_nodiag(Gv, deg.p, st);
  CK(cudaMemsetAsync(level.p, 0xFF, n1 * sizeof(int32_t), st));  // -1: unvisited
  CK(cudaMemsetAsync(done.p, 0, n1, st));
  // components of G on the host (one copy of G's pattern); their order is that of their
  // smallest (degree, index) node.  Components of up to kRcmHost nodes (isolated nodes,
  // the many small clusters of a sparse graph) are ordered on the host by the same rules --
  // each would cost the device loop a dozen launches and syncs per BFS level -- the large
  // ones on the device.
  constexpr int64_t kRcmHost = 4096;
  std::vector<int64_t> hrp((size_t)n + 1);
  std::vector<int32_t> hcol((size_t)std::max<int64_t>(G.nnz, 1)), hdeg(n1);
  CK(cudaMemcpyAsync(hrp.data(), G.rp.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (G.nnz) CK(cudaMemcpyAsync(hcol.data(), G.col.p, G.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hdeg.data(), deg.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int32_t> comp(n1, -1), cnodes;  // component id; nodes grouped by component
  std::vector<int64_t> cstart, cmin;           // start of each component in cnodes; min key
  cnodes.reserve((size_t)n);
  for (int64_t v0 = 0; v0 < n; v0++) {
    if (comp[v0] >= 0) continue;
    const int32_t c = (int32_t)cstart.size();
    cstart.push_back((int64_t)cnodes.size());
    int64_t mk = INT64_MAX;
    size_t head = cnodes.size();
    cnodes.push_back((int32_t)v0);
    comp[v0] = c;
    while (head < cnodes.size()) {
      const int32_t v = cnodes[head++];
      mk = std::min<int64_t>(mk, ((int64_t)hdeg[v] << 32) | v);
      for (int64_t p = hrp[v]; p < hrp[v + 1]; p++) {
        const int32_t u = hcol[p];
        if (u != v && comp[u] < 0) {
          comp[u] = c;
          cnodes.push_back(u);
        }
      }
    }
    cmin.push_back(mk);
  }
  const int64_t ncomp = (int64_t)cstart.size();
  cstart.push_back((int64_t)cnodes.size());
  std::vector<int64_t> corder((size_t)ncomp);
  for (int64_t c = 0; c < ncomp; c++) corder[c] = c;
  std::sort(corder.begin(), corder.end(), [&](int64_t a, int64_t b) { return cmin[a] < cmin[b]; });
  std::vector<int64_t> hcm((size_t)n1), hpos(n1);
  std::vector<int32_t> hlev(n1, -1);
  std::vector<int32_t> q;
  auto hbfs = [&](int32_t s, std::vector<int64_t> &lo) -> int {  // host BFS levels of s
    q.clear();
    q.push_back(s);
    hlev[s] = 0;
    lo.assign({0});
    size_t head = 0;
    int cur = 0;
    while (head < q.size()) {
      const int32_t v = q[head++];
      if (hlev[v] != cur) {
        cur = hlev[v];
        lo.push_back((int64_t)head - 1);
      }
      for (int64_t p = hrp[v]; p < hrp[v + 1]; p++) {
        const int32_t u = hcol[p];
        if (u != v && hlev[u] < 0) {
          hlev[u] = hlev[v] + 1;
          q.push_back(u);
        }
      }
    }
    lo.push_back((int64_t)q.size());
    return (int)lo.size() - 1;
  };
  auto hreset = [&]() {
    for (int32_t v : q) hlev[v] = -1;
  };
  std::vector<int64_t> hlo;
  std::vector<std::pair<int64_t, int64_t>> large;  // (component, base) done on the device
  int64_t base = 0;
  for (int64_t ci = 0; ci < ncomp; ci++) {
    const int64_t c = corder[ci], size = cstart[c + 1] - cstart[c];
    if (size > kRcmHost) {
      large.push_back({c, base});
      base += size;
      continue;
    }
    int32_t s0 = (int32_t)(cmin[c] & 0xFFFFFFFF);
    int nl = hbfs(s0, hlo);
    for (;;) {  // George-Liu pseudo-peripheral node
      int32_t cnd = -1;
      for (int64_t t = hlo[nl - 1]; t < hlo[nl]; t++) {
        const int32_t v = q[t];
        if (cnd < 0 || hdeg[v] < hdeg[cnd] || (hdeg[v] == hdeg[cnd] && v < cnd)) cnd = v;
      }
      hreset();
      const int nl2 = hbfs(cnd, hlo);
      if (nl2 > nl) {
        s0 = cnd;
        nl = nl2;
      } else {
        hreset();
        nl = hbfs(s0, hlo);
        break;
      }
    }
    // Cuthill-McKee over the levels: (smallest position of a neighbour one level up,
    // degree, index)
    std::vector<std::tuple<int64_t, int32_t, int32_t>> lv;
    hcm[base] = s0;
    hpos[s0] = base;
    for (int L = 1; L < nl; L++) {
      lv.clear();
      for (int64_t t = hlo[L]; t < hlo[L + 1]; t++) {
        const int32_t v = q[t];
        int64_t k = INT64_MAX;
        for (int64_t p = hrp[v]; p < hrp[v + 1]; p++) {
          const int32_t u = hcol[p];
          if (u != v && hlev[u] == L - 1) k = std::min(k, hpos[u]);
        }
        lv.emplace_back(k, hdeg[v], v);
      }
      std::sort(lv.begin(), lv.end());
      for (size_t t = 0; t < lv.size(); t++) {
        const int32_t v = std::get<2>(lv[t]);
        hcm[base + hlo[L] + (int64_t)t] = v;
        hpos[v] = base + hlo[L] + (int64_t)t;
      }
    }
    hreset();
    base += size;
  }
  std::vector<int64_t> loff;
  auto bfs = [&](int64_t s) -> int {  // levels from s; loff = level boundaries in queue
    const int32_t zero = 0;
    CK(cudaMemcpyAsync(level.p + s, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(queue.p, &s, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const unsigned long long one = 1;
    CK(cudaMemcpyAsync(tail.p, &one, sizeof(one), cudaMemcpyHostToDevice, st));
    loff.assign({0, 1});
    int64_t a = 0, b = 1;
    for (int32_t L = 0; b > a; L++) {
      launch_bfs_expand(Gv, queue.p, a, b, level.p, L, tail.p, st);
      const int64_t nb = (int64_t)d2h(tail.p, st);
      a = b;
      b = nb;
      if (b > a) loff.push_back(b);
    }
    return (int)loff.size() - 1;
  };
  auto argmin = [&](const int64_t *qq, int64_t a, int64_t b, const int8_t *dn) -> int64_t {
    const unsigned long long init = ~0ull;
    CK(cudaMemcpyAsync(mn.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    launch_min_deg(qq, a, b, deg.p, dn, mn.p, st);
    return (int64_t)(d2h(mn.p, st) & 0xFFFFFFFFull);
  };
  for (auto &cb : large) {  // the large components on the device
    const int64_t placed = cb.second;
    int64_t s = (int64_t)(cmin[cb.first] & 0xFFFFFFFF);
    int nl = bfs(s);
    for (;;) {  // George-Liu pseudo-peripheral node
      const int64_t c = argmin(queue.p, loff[nl - 1], loff[nl], nullptr);
      const int64_t qlen = loff[nl];
      launch_reset_level(queue.p, 0, qlen, level.p, st);
      const int nl2 = bfs(c);
      if (nl2 > nl) {
        s = c;
        nl = nl2;
      } else {
        launch_reset_level(queue.p, 0, loff[nl2], level.p, st);
        nl = bfs(s);
        break;
      }
    }
    const int64_t qlen = loff[nl];
    CK(cudaMemcpyAsync(pos.p + s, &placed, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(cm.p + placed, &s, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    for (int L = 1; L < nl; L++) {
      const int64_t a = loff[L], b = loff[L + 1];
      launch_cm_key(Gv, queue.p, a, b, level.p, L - 1, pos.p, deg.p, key.p, ids.p, st);
      launch_cm_sort_place(key.p, ids.p, b - a, key2.p, ids2.p, keyv.p, tmp.p, tb, placed + a, pos.p,
                           cm.p, st);
    }
    launch_mark_done(cm.p, placed, placed + qlen, done.p, level.p, st);
    // the device's segment into the host order
    CK(cudaMemcpyAsync(hcm.data() + placed, cm.p + placed, qlen * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemcpyAsync(cm.p, hcm.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  perm.ensure(n1, st);
  inv.ensure(n1, st);
  launch_reverse_perm(cm.p, n, perm.p, inv.p, st);
  CK(cudaStreamSynchronize(st));
}

static void do_plan(sexpm_plan_s &P, const sexpm_csr_in *H, double eps_tol) {
  cudaStream_t st = P.st;
  REQUIRE(H->n >= 1, SEXPM_EINVAL, "n must be >= 1");
  REQUIRE(H->row_begin >= 0 && H->row_end <= H->n && H->row_begin <= H->row_end, SEXPM_EINVAL,
          "bad row range");
  REQUIRE(H->n < INT32_MAX, SEXPM_EINVAL, "n must fit int32 column indices");
  REQUIRE(H->nnz >= 0 && (H->nnz == 0 || (H->colidx && H->vals)) && H->rowptr, SEXPM_EINVAL,
          "null CSR arrays");
  REQUIRE(isfinite(eps_tol) && eps_tol >= 1e-16, SEXPM_ETOL,
          "eps_tol must be >= 1e-16 (unit roundoff, reading R13)");
  REQUIRE(P.o.e_r > 0.0, SEXPM_EINVAL, "e_r must be > 0");
  P.n = H->n;
  P.row_begin = H->row_begin;
  P.row_end = H->row_end;
  P.eps_tol = eps_tol;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  const bool plog = getenv("SEXPM_PLAN_LOG") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto mark = [&](const char *what) {  // SEXPM_PLAN_LOG: host-side phase times of the plan
    if (!plog) return;
    CK(cudaStreamSynchronize(st));
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[sexpm plan] %-28s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(t - tprev).count());
    tprev = t;
  };
  Workspace &w = P.ws;
  w.flags.ensure(1, st);
  w.partial.ensure(1024, st);
  w.scal.ensure(8, st);
  // validate the local block
  CsrView L = view_of(H);
  CK(cudaMemsetAsync(w.flags.p, 0, sizeof(int), st));
  int64_t rp01[2];
  CK(cudaMemcpyAsync(&rp01[0], L.rp, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rp01[1], L.rp + L.nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  mark("input + rowptr ends");
  REQUIRE(rp01[0] == 0 && rp01[1] == L.nnz, SEXPM_EINVAL, "rowptr[0] must be 0 and rowptr[rows] == nnz");
  launch_validate(L, P.n, w.flags.p, st);
  int vf = d2h(w.flags.p, st);
  vf = (int)allmax(P, (double)vf);
  REQUIRE(!(vf & 8), SEXPM_ENONFINITE, "H holds a non-finite value");
  REQUIRE(!(vf & 7), SEXPM_EINVAL, "malformed CSR (rowptr / column range / column order)");
  mark("validate");
  sexpm_csr_in Hp_in;
  if (P.o.reorder) {  // N3: work on P H P^T (RCM order); do_run maps E back
    REQUIRE(P.world == 1, SEXPM_EINVAL, "reorder is single-GPU (the RCM needs all of H)");
    compute_rcm(P, L, P.perm, P.inv);
    permute_csr(P, L, P.perm.p, P.inv.p, P.Hperm);  // row i <- row perm[i], col c -> inv[c]
    Hp_in = *H;
    Hp_in.rowptr = P.Hperm.rp.p;
    Hp_in.colidx = P.Hperm.col.p;
    Hp_in.vals = P.Hperm.val.p;
    H = &Hp_in;
    L = view_of(H);
    mark("reorder (RCM)");
  }
  // rank partition
  std::vector<double> rb;
  double mine[2] = {(double)P.row_begin, (double)P.row_end};
  gather_doubles(P, mine, 2, rb);
  P.bounds.assign(P.world + 1, 0);
  for (int g = 0; g < P.world; g++) {
    REQUIRE((int64_t)rb[2 * g] == (g == 0 ? 0 : (int64_t)rb[2 * g - 1]), SEXPM_EINVAL,
            "row blocks must be contiguous in rank order");
    P.bounds[g + 1] = (int64_t)rb[2 * g + 1];
  }
  REQUIRE(P.bounds[P.world] == P.n, SEXPM_EINVAL, "row blocks must cover [0, n)");
  // full H on every rank (explicit zeros purged: compaction with tau = 0)
  DCsr Hraw;
  if (P.world == 1) {
    copy_csr(P, L, Hraw);
  } else {
    allgather_rows(P, L, Hraw);
  }
  {
    w.row_off.ensure((size_t)P.n, st);
    w.row_cnt.ensure((size_t)P.n, st);
    w.cnt.ensure((size_t)P.n, st);
    w.scan_tmp.ensure((size_t)scan_tmp_elems(P.n) + 1, st);
    // row_off = rp[0..n), row_cnt = rp diff
    launch_copy_i64_offset(Hraw.rp.p, P.n, 0, w.row_off.p, st);
    launch_row_lengths(Hraw.rp.p, P.n, w.row_cnt.p, st);
    launch_compact_count(P.n, w.row_off.p, w.row_cnt.p, Hraw.val.p, 0.0, w.cnt.p, st);
    DCsr Hc;
    Hc.nrows = P.n;
    Hc.row0 = 0;
    Hc.rp.alloc((size_t)P.n + 1, st);
    launch_exclusive_scan(w.cnt.p, P.n, Hc.rp.p, w.scan_tmp.p, st);
    Hc.nnz = d2h(Hc.rp.p + P.n, st);
    Hc.col.alloc((size_t)Hc.nnz, st);
    Hc.val.alloc((size_t)Hc.nnz, st);
    launch_compact_write(P.n, 0, w.row_off.p, w.row_cnt.p, Hraw.col.p, Hraw.val.p, 0.0, Hc.rp.p,
                         Hc.col.p, Hc.val.p, nullptr, nullptr, nullptr, st);
    P.H0full = std::move(Hc);
  }
  DCsr &Hf = P.H0full;
  mark("gather + purge zeros");
  // K8 norms on the device
  double norm = 0.0;
  int symflags = 3;
  {
    DCsr HT;
    build_transpose(P, Hf.view(), P.n, HT);
    DBuf<int64_t> &cp = HT.rp;
    DBuf<int32_t> &trow = HT.col;
    DBuf<double> &tval = HT.val;
    DBuf<double> colsum;
    if (P.o.plan_norm == 0) {
      colsum.alloc((size_t)P.n, st);
      launch_col_abs_sum(P.n, cp.p, tval.p, colsum.p, st);
      launch_reduce_max(colsum.p, P.n, w.partial.p, w.scal.p, st);
    } else {
      launch_reduce_sumsq(Hf.val.p, Hf.nnz, w.partial.p, w.scal.p, st);
    }
    CK(cudaMemsetAsync(w.flags.p, 0, sizeof(int), st));
    launch_compare_transpose(Hf.view(), cp.p, trow.p, tval.p, w.flags.p, st);
    double s = d2h(w.scal.p, st);
    norm = P.o.plan_norm == 0 ? s : sqrt(s);
    if (Hf.nnz == 0) norm = 0.0;
    symflags = d2h(w.flags.p, st);
    // keep the transpose: H0^T (scaled below) feeds the Taylor pull kernel
    P.H0T = std::move(HT);
  }
  mark("transpose + norm + symmetry");
  P.norm = norm;
  int M, N;
  REQUIRE(select_MN(norm, eps_tol, P.o.m_cap, P.o.n_window, M, N), SEXPM_EINFEASIBLE,
          "Eq. (4.20) infeasible within m_cap / n_window");
  if (P.o.force_M >= 0) M = P.o.force_M;
  if (P.o.force_N >= 0) N = P.o.force_N;
  P.M = M;
  P.N = N;
  int normal = P.o.normal;
  if (normal < 0) normal = ((symflags & 1) == 0) || ((symflags & 2) == 0);
  P.h_sym = (symflags & 1) == 0;
  P.normal = normal;
  filter_budgets(norm, normal, M, N, P.a, P.r0, P.eps_g0);
  if (!P.o.filter) P.eps_g0 = 0.0;
  // H0 = H 2^-N (exact)
  launch_scale_pow2(Hf.val.p, Hf.nnz, -N, st);
  launch_scale_pow2(P.H0T.val.p, P.H0T.nnz, -N, st);
  mark("plan (M,N) + scale");
  build_diagonals(P);
  build_window(P);
  mark("diagonals");
  slice_rows(P, Hf, P.row_begin, P.row_end, P.H0loc);
  // The squarings' processing order (locality clusters of H's graph, host BFS) is computed
  // on a background host thread with its own stream, overlapping the Taylor phase on the
  // GPU; sexpm_run waits for it (event) before the first squaring.
  {
    const int64_t nl = P.row_end - P.row_begin;
    P.proc_order.ensure((size_t)std::max<int64_t>(nl, 1), st);
    P.block_order.ensure((size_t)std::max<int64_t>((nl + 7) / 8, 1), st);
    if (P.o.sq_order == 1 && P.N >= 1) {
      P.tperm.ensure((size_t)std::max<int64_t>(P.n, 1), st);
      P.tinv.ensure((size_t)std::max<int64_t>(P.n, 1), st);
      P.tperm_loc.ensure((size_t)std::max<int64_t>(nl, 1), st);
      P.tinv_loc.ensure((size_t)std::max<int64_t>(nl, 1), st);
      P.block_order_t.ensure((size_t)std::max<int64_t>((P.n + 7) / 8, 1), st);
    }
    LatticeDesc Ld;
    if (P.world == 1 && P.o.sq_order == 1 && P.N >= 1 && !P.o.ssat && P.M >= 1 && detect_lattice(P, Ld)) {
      // grid stencil on one GPU: the aggregate order is arithmetic, computed on the device
      // (no host thread, no pattern download); row / block orders of the untiled kernels =
      // index order
      DBuf<unsigned> mask;
      DBuf<int64_t> cnt, off;
      DBuf<int32_t> key, scnt, cur;
      DBuf<int> flag;
      const int64_t nbt = (P.n + 7) / 8, big = std::max(std::max(2 * (Ld.ntiles + 1), Ld.nsuper + 1), nbt);
      mask.alloc((size_t)Ld.ntiles, st);
      cnt.alloc((size_t)big, st);
      off.alloc((size_t)big, st);
      key.alloc((size_t)nbt, st);
      scnt.alloc((size_t)Ld.nsuper, st);
      cur.alloc((size_t)Ld.nsuper, st);
      flag.alloc(1, st);
      w.scan_tmp.ensure((size_t)scan_tmp_elems(big) + 1, st);
      launch_lattice_order(Ld, mask.p, cnt.p, off.p, w.scan_tmp.p, key.p, scnt.p, cur.p, flag.p, P.tperm.p,
                           P.tinv.p, P.block_order_t.p, st);
      REQUIRE(d2h(flag.p, st) == 0, SEXPM_EINTERNAL, "lattice order: a supertile holds more block rows than the segment sort");
      CK(cudaMemcpyAsync(P.tperm_loc.p, P.tperm.p, P.n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(P.tinv_loc.p, P.tinv.p, P.n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      launch_iota_i32(nl, P.proc_order.p, st);
      launch_iota_i32((nl + 7) / 8, P.block_order.p, st);
      CK(cudaStreamSynchronize(st));  // the scratch buffers are local
      P.tperm_ready = true;
      P.agg_kind = Ld.dims == 2 ? 3 : 4;
      P.order_pending = false;
      mark("lattice order (device)");
    } else if (P.dia_nd > 0 && std::max<int64_t>(-(int64_t)P.dia_dmin, (int64_t)P.dia_dmax) <= 4) {
      // a band of half-width <= 4 (1D stencils) is best in index order: no host ordering
      launch_iota_i32(nl, P.proc_order.p, st);
      launch_iota_i32((nl + 7) / 8, P.block_order.p, st);
      mark("index order (narrow band)");
    } else {
    CK(cudaEventCreateWithFlags(&P.ev_pattern, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&P.ev_order, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&P.bg_st, cudaStreamNonBlocking));
    CK(cudaEventRecord(P.ev_pattern, st));
    P.order_pending = true;
    P.bg = std::thread([&P]() {
      const auto b0 = std::chrono::steady_clock::now();
      try {
        CK(cudaSetDevice(P.dev));
        CK(cudaStreamWaitEvent(P.bg_st, P.ev_pattern, 0));
        const DCsr &F = P.H0full;
        std::vector<int64_t> hrp((size_t)P.n + 1);
        std::vector<int32_t> hcol((size_t)std::max<int64_t>(F.nnz, 1));
        CK(cudaMemcpyAsync(hrp.data(), F.rp.p, hrp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, P.bg_st));
        if (F.nnz)
          CK(cudaMemcpyAsync(hcol.data(), F.col.p, F.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, P.bg_st));
        CK(cudaStreamSynchronize(P.bg_st));
        auto lap = [&](const char *what) {
          if (getenv("SEXPM_PLAN_LOG"))
            fprintf(stderr, "[sexpm order] %-28s %8.1f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - b0).count());
        };
        lap("pattern D2H");
        std::vector<int32_t> &ord = P.h_order;
        // the cluster order of this rank's rows runs on its own host thread, beside the
        // aggregate candidates below
        std::thread t_clu([&] { cluster_order(hrp, hcol, P.row_begin, P.row_end, 1024, ord); });
        // the aggregate order: for every rank range whose rows can be columns of this rank's
        // T^_0 rows (within M x H's bandwidth, Lemma 3.1), both candidates built and judged
        // on that range alone (so every rank takes the same decision for a range)
        const bool want_agg = P.o.sq_order == 1 && P.N >= 1;
        std::vector<std::vector<int64_t>> range_perm;
        std::vector<int> range_kind;
        std::vector<int> needed;
        std::vector<int64_t> range_blocks;  // per needed range: sampled blocks idx, BFS, compact
        if (want_agg) {
          int64_t lH = 0;
          for (int64_t r = 0; r < P.n; r++)
            if (hrp[r + 1] > hrp[r])
              lH = std::max<int64_t>(lH, std::max<int64_t>(std::llabs((int64_t)hcol[hrp[r]] - r),
                                                           std::llabs((int64_t)hcol[hrp[r + 1] - 1] - r)));
          // columns of this rank's iterates, and of the halo rows it receives, stay within
          // 2^(N+1) M l(H) of its rows (Lemma 3.1: l(T^_0) <= M l(H), each squaring at most
          // doubles it, a halo row is within l(T^_{i-1}) of the range)
          const int64_t reach = (int64_t)std::min<double>((double)P.n, std::ldexp((double)std::max(P.M, 1) * (double)lH, P.N + 1));
          const int64_t wlo = std::max<int64_t>(0, P.row_begin - reach), whi = std::min<int64_t>(P.n, P.row_end + reach);
          for (int g = 0; g < P.world; g++)
            if (P.bounds[g] < whi && P.bounds[g + 1] > wlo && P.bounds[g + 1] > P.bounds[g]) needed.push_back(g);
          range_perm.assign(needed.size(), {});
          range_kind.assign(needed.size(), 0);
          range_blocks.assign(needed.size() * 3, 0);
          const int rad = std::max(3, std::min(16, (int)lround(0.8 * P.M)));
          std::vector<std::thread> ts;
          for (size_t q = 0; q < needed.size(); q++)
            ts.emplace_back([&, q] {
              const int g = needed[q];
              const int64_t lo = P.bounds[g], hi = P.bounds[g + 1];
              // judged on a window of <= 2^16 rows in the middle of the range (8-aligned),
              // then only the chosen candidate is built for the whole range
              const int64_t wn = std::min<int64_t>(hi - lo, 65536);
              const int64_t wlo = std::min<int64_t>(hi - wn, lo + (((hi - lo - wn) / 2) & ~(int64_t)7));
              const int64_t whi = wlo + wn;
              std::vector<int64_t> cb, cc;
              std::thread tb([&] { aggregate_order(hrp, hcol, wlo, whi, 8, cb); });
              aggregate_order_compact(hrp, hcol, wlo, whi, 8, cc);
              tb.join();
              int64_t bl[3];
              std::thread p0([&] { bl[0] = sampled_blocks(hrp, hcol, wlo, whi, nullptr, rad); });
              std::thread p1([&] { bl[1] = sampled_blocks(hrp, hcol, wlo, whi, &cb, rad); });
              bl[2] = sampled_blocks(hrp, hcol, wlo, whi, &cc, rad);
              p0.join();
              p1.join();
              const int pick = bl[2] < bl[1] ? 1 : 0;
              const int64_t b_agg = pick ? bl[2] : bl[1];
              for (int k = 0; k < 3; k++) range_blocks[3 * q + k] = bl[k];
              if (10 * b_agg <= 9 * bl[0]) {
                if (wlo == lo && whi == hi) {
                  range_perm[q].swap(pick ? cc : cb);
                } else if (pick) {
                  aggregate_order_compact(hrp, hcol, lo, hi, 8, range_perm[q]);
                } else {
                  aggregate_order(hrp, hcol, lo, hi, 8, range_perm[q]);
                }
                range_kind[q] = 1 + pick;
              }
            });
          for (auto &t : ts) t.join();
        }
        t_clu.join();
        lap("cluster order + aggregates");
        // block rows (8 rows) of the block kernel, in the order their first row appears
        std::vector<int32_t> &bo = P.h_border;
        bo.clear();
        {
          std::vector<uint8_t> seenb((ord.size() + 7) / 8 + 1, 0);
          for (int32_t r : ord) {
            const int32_t I = r >> 3;
            if (!seenb[I]) {
              seenb[I] = 1;
              bo.push_back(I);
            }
          }
        }
        if (!bo.empty())
          CK(cudaMemcpyAsync(P.block_order.p, bo.data(), bo.size() * sizeof(int32_t), cudaMemcpyHostToDevice, P.bg_st));
        if (!ord.empty())
          CK(cudaMemcpyAsync(P.proc_order.p, ord.data(), ord.size() * sizeof(int32_t), cudaMemcpyHostToDevice, P.bg_st));
        if (want_agg) {
          // assemble the global permutation: each needed range relabelled within itself,
          // identity elsewhere (those labels never occur in this rank's data)
          P.h_tperm.clear();
          P.agg_kind = 0;
          bool any = false;
          for (size_t q = 0; q < needed.size(); q++) {
            if (getenv("SEXPM_PLAN_LOG"))
              fprintf(stderr, "[sexpm plan] aggregate order, rows [%lld, %lld): sampled blocks index %lld, BFS %lld, compact %lld -> %s\n",
                      (long long)P.bounds[needed[q]], (long long)P.bounds[needed[q] + 1], (long long)range_blocks[3 * q],
                      (long long)range_blocks[3 * q + 1], (long long)range_blocks[3 * q + 2],
                      range_kind[q] == 0 ? "index order" : (range_kind[q] == 1 ? "BFS" : "compact"));
            if (range_kind[q]) any = true;
            if (needed[q] == P.rank) P.agg_kind = range_kind[q];
          }
          std::vector<int64_t> hinv;
          if (any) {
            P.h_tperm.resize((size_t)P.n);
            for (int64_t i = 0; i < P.n; i++) P.h_tperm[i] = i;
            for (size_t q = 0; q < needed.size(); q++)
              if (range_kind[q])
                std::copy(range_perm[q].begin(), range_perm[q].end(), P.h_tperm.begin() + P.bounds[needed[q]]);
            hinv.resize((size_t)P.n);
            for (int64_t i = 0; i < P.n; i++) hinv[P.h_tperm[i]] = i;
          }
          // block rows of the relabelled matrix in the locality order of H's clusters: each
          // aggregate ranked by the earliest position of its rows in `ord`
          if (!P.h_tperm.empty() && P.world == 1) {
            std::vector<int32_t> at((size_t)P.n);
            for (size_t j = 0; j < ord.size(); j++) at[ord[j]] = (int32_t)j;
            const int64_t nbt = (P.n + 7) / 8;
            std::vector<std::pair<int32_t, int32_t>> key((size_t)nbt);
            for (int64_t g = 0; g < nbt; g++) {
              int32_t k = INT32_MAX;
              for (int64_t i = 8 * g; i < std::min<int64_t>(P.n, 8 * g + 8); i++) k = std::min(k, at[P.h_tperm[i]]);
              key[g] = {k, (int32_t)g};
            }
            std::sort(key.begin(), key.end());
            std::vector<int32_t> bot((size_t)nbt);
            for (int64_t g = 0; g < nbt; g++) bot[g] = key[g].second;
            CK(cudaMemcpyAsync(P.block_order_t.p, bot.data(), nbt * sizeof(int32_t), cudaMemcpyHostToDevice, P.bg_st));
            CK(cudaStreamSynchronize(P.bg_st));  // bot is local
          }
          if (!P.h_tperm.empty()) {
            // this rank's rows: local old row of local new row i, and the inverse
            const int64_t rb = P.row_begin, nloc = P.row_end - P.row_begin;
            std::vector<int64_t> ploc((size_t)std::max<int64_t>(nloc, 1)), iloc((size_t)std::max<int64_t>(nloc, 1));
            for (int64_t i = 0; i < nloc; i++) {
              ploc[i] = P.h_tperm[rb + i] - rb;
              iloc[i] = hinv[rb + i] - rb;
            }
            CK(cudaMemcpyAsync(P.tperm.p, P.h_tperm.data(), P.n * sizeof(int64_t), cudaMemcpyHostToDevice, P.bg_st));
            CK(cudaMemcpyAsync(P.tinv.p, hinv.data(), P.n * sizeof(int64_t), cudaMemcpyHostToDevice, P.bg_st));
            CK(cudaMemcpyAsync(P.tperm_loc.p, ploc.data(), nloc * sizeof(int64_t), cudaMemcpyHostToDevice, P.bg_st));
            CK(cudaMemcpyAsync(P.tinv_loc.p, iloc.data(), nloc * sizeof(int64_t), cudaMemcpyHostToDevice, P.bg_st));
            CK(cudaStreamSynchronize(P.bg_st));  // host vectors are local
            P.tperm_ready = true;
          }
        }
        lap("done");
        CK(cudaEventRecord(P.ev_order, P.bg_st));
        P.order_host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - b0).count();
      } catch (const SxError &e) {
        P.bg_err = e.msg.empty() ? "order thread failed" : e.msg;
      } catch (...) {
        P.bg_err = "order thread failed";
      }
    });
    }
  }
  mark("groups + upload");
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaEventElapsedTime(&P.plan_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// ------------------------------------------------------------------------------------
// run: Taylor phase, squarings, finish
// ------------------------------------------------------------------------------------
static void swap_csr(DCsr &a, DCsr &b) {
  DCsr t = std::move(a);
  a = std::move(b);
  b = std::move(t);
}

// Taylor phase on the offset window K5w (Alg. 4.2 step 3): one launch per term
// i = 2..M (S~_i from the checkpoint of S~_{i-1}, T^_0^(i-1) accumulated on the way), the
// Algorithm 4.1 passes over the staged band values, then T^_0 = T^_0^(m-1) + S^_m
// (m = M_eff) written as CSR (count, scan, write).  Returns M_eff.
static int taylor_window(sexpm_plan_s &P, DCsr &T, const std::function<double()> &step_ms,
                         cudaEvent_t a0) {
  auto &W = P.win;
  Workspace &w = P.ws;
  cudaStream_t st = P.st;
  sexpm_stats &S = P.stats;
  const auto h_start = std::chrono::steady_clock::now();
  const int64_t nl = P.row_end - P.row_begin;
  const size_t nl1 = (size_t)std::max<int64_t>(nl, 1);
  int maxl = 1, maxc = 1, maxlp = 1;
  for (int j = 1; j <= P.M; j++) {
    maxl = std::max(maxl, W.lcnt[j]);
    maxc = std::max(maxc, W.ccnt[j]);
    maxlp = std::max(maxlp, W.half ? W.lcnt_h[j] : W.lcnt[j]);
  }
  // half window (symmetric path): planes over the offsets o >= 0, padr zero rows in front
  const int64_t plane = nl + W.padr;
  const int nUs = W.half ? W.nUh : W.nU;
  auto lc = [&](int j) { return W.half ? W.lcnt_h[j] : W.lcnt[j]; };
  DBuf<double> *ck_s[2] = {&P.Tn.val, &P.E.val};
  DBuf<double> &t0buf = w.bsrB.bval;
  // one extra (zero) plane each: the records' "absent" operand
  if (P.M >= 2)
    for (int k = 0; k < 2; k++) {
      ck_s[k]->ensure((size_t)std::max<int64_t>(plane, 1) * (size_t)(maxlp + 1), st);
      if (W.padr > 0)  // the pad rows stay zero: the kernels never write them
        CK(cudaMemset2DAsync(ck_s[k]->p, (size_t)plane * sizeof(double), 0, (size_t)W.padr * sizeof(double),
                             (size_t)(maxlp + 1), st));
    }
  t0buf.ensure(nl1 * (size_t)(nUs + 1), st);
  CK(cudaMemsetAsync(t0buf.p + (size_t)nUs * nl, 0, nl1 * sizeof(double), st));
  // band values staged in the staging pool (position-major, band_cap per row)
  // (a row of S~_i has at most |W_i| <= maxl values: sized for that, no term ever re-runs; the
  // pool is the squarings' staging pool, which is larger anyway)
  int64_t band_cap = maxl;
  if (getenv("SEXPM_WIN_BAND")) band_cap = std::max<int64_t>(1, atoll(getenv("SEXPM_WIN_BAND")));  // debug: initial band slots
  w.row_cnt.ensure(nl1, st);
  w.row_nnz.ensure(nl1, st);
  w.row_fsum.ensure(nl1, st);
  w.row_p1.ensure(nl1, st);
  w.row_c1.ensure(nl1, st);
  w.passrow.ensure(nl1, st);
  w.cnt.ensure(nl1, st);
  w.cnt2.ensure(nl1, st);
  w.scan_tmp.ensure((size_t)scan_tmp_elems(nl) + 1, st);
  w.partial.ensure(1024, st);
  w.scal.ensure(8, st);
  w.i64tmp.ensure(8, st);
  WinArgs base;
  base.nrows = nl;
  base.row0 = P.row_begin;
  base.n = P.n;
  base.nd = P.dia_nd;
  base.dia = P.dia_val.p;
  base.doff = P.dia_off.p;
  base.dzero = W.dzero;
  base.dpad = W.dpad.p + W.pad;
  base.hpad = (int32_t)W.pad;
  for (int di = 0; di < kDiaMax; di++)
    base.hoff[di] = di < P.dia_nd ? (int32_t)((int64_t)di * W.npad - P.h_dia_off[di]) : 0;
  base.row_cnt = w.row_cnt.p;
  base.row_nnz = w.row_nnz.p;
  base.row_c1 = w.row_c1.p;
  base.row_fsum = w.row_fsum.p;
  base.row_p1 = w.row_p1.p;
  base.half = W.half ? 1 : 0;
  base.plane = plane;
  base.padr = W.padr;
  // CTAs (4 warps) per SM of the term kernel (default: one CTA per tile of 128 rows)
  const int win_ctas = getenv("SEXPM_WIN_CTAS") ? std::max(1, atoi(getenv("SEXPM_WIN_CTAS"))) : 1 << 20;
  cudaEvent_t k0, k1;
  CK(cudaEventCreate(&k0));
  CK(cudaEventCreate(&k1));
  int sa = 0;  // ck_s[sa] = S~_{i-1}
  double tau_prev = 0.0;
  int64_t prev_nnz_local = 0;
  bool t0_complete = false;
  int M_eff = 1;
  if (getenv("SEXPM_STEP_LOG")) CK(cudaStreamSynchronize(st));
  const auto h_loop = std::chrono::steady_clock::now();
  const double eps_g = P.eps_g0;
  for (int i = 2; i <= P.M; i++) {
    CK(cudaEventRecord(a0, st));
    WinArgs a = base;
    a.prev_is_h0 = i == 2;
    a.pS = ck_s[sa]->p;
    a.tau_prev = tau_prev;
    a.T0old = t0buf.p;  // in place
    a.T0new = t0buf.p;
    a.c1cnt = W.ccnt[i - 1];
    a.mapC = W.mapC.p + W.coff[i - 1];
    a.mapW = W.mapW.p + W.coff[i - 1];
    a.cumU = W.cumU.p + W.coff[i - 1];
    a.ncnt = lc(i);
    a.rec = W.rec.p + W.woff[i];
    a.nS = ck_s[sa ^ 1]->p;
    // zero planes of the inputs (absent operands)
    if (i > 2) CK(cudaMemsetAsync(ck_s[sa]->p + (size_t)lc(i - 1) * plane, 0, (size_t)plane * sizeof(double), st));
    if (W.dzero < 0) launch_taylor_win_t0(a, st);  // T^_0 update not fused
    a.divisor = (double)i;
    // floor lemma: K = n |W_i| bounds the entries of S~_i
    const double K = (double)P.n * (double)W.lcnt[i];
    a.floor_tau = (eps_g > 0.0 && K > 0.0) ? eps_g / sqrt(K) : 0.0;
    a.eps_g = eps_g;
    // band staging sized from the previous terms; re-run once at the size a row needed (the
    // launch is idempotent: its outputs never alias its inputs)
    for (int attempt = 0;; attempt++) {
      w.pool_val.ensure(nl1 * (size_t)band_cap, st);
      w.pool_col.ensure(nl1 * (size_t)band_cap, st);
      a.band_val = w.pool_val.p;
      a.band_col = w.pool_col.p;
      a.band_cap = band_cap;
      a.band_need = W.need.p;
      CK(cudaMemsetAsync(W.need.p, 0, sizeof(unsigned long long), st));
      CK(cudaEventRecord(k0, st));
      launch_taylor_win(a, win_ctas, P.sm_count, st);
      CK(cudaGetLastError());
      CK(cudaEventRecord(k1, st));
      const unsigned long long need = d2h(W.need.p, st);
      if (need == 0) break;
      REQUIRE(attempt < 2, SEXPM_EINTERNAL, "window Taylor kernel: band staging keeps overflowing");
      band_cap = std::min<int64_t>(maxl, (int64_t)need + need / 4 + 16);
      P.retries++;
    }
    // Algorithm 4.1 over the band values
    launch_reduce_sum(w.row_fsum.p, nl, w.partial.p, w.scal.p + 0, st);
    launch_reduce_sum(w.row_p1.p, nl, w.partial.p, w.scal.p + 3, st);
    launch_reduce_sum_i64(w.row_nnz.p, nl, w.i64tmp.p + 3, st);
    launch_reduce_sum_i64(w.row_c1.p, nl, w.i64tmp.p + 4, st);
    launch_reduce_sum_i64(w.row_cnt.p, nl, w.i64tmp.p + 5, st);
    double hs[4];
    int64_t hi[3];
    // products with a nonzero left operand: nd per entry of S^_{i-1} (h may be 0 at a boundary)
    const double prods = (double)P.dia_nd * (double)(i == 2 ? P.H0loc.nnz : prev_nnz_local);
    CK(cudaMemcpyAsync(hs, w.scal.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hi, w.i64tmp.p + 3, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double F = allsum(P, hs[0]);
    int passes = 0;
    double tau = 0.0;
    if (eps_g > 0.0) {
      // m_0 = 1; the first pass always runs (reading R1; tau_1 = eps_g: fused), then the
      // passes repeat while b_n > eps_g (1 + e_r)
      long double m = 1.0L, b = INFINITY;
      const long double eg = eps_g, lim = eg * (1.0L + (long double)P.o.e_r);
      long double epsf = INFINITY;
      while (passes == 0 || b > lim) {
        epsf = eg / m;
        const double tau_d = (double)epsf;
        double Sp;
        if (passes == 0 && tau_d == eps_g) {
          Sp = allsum(P, hs[3]);
        } else {
          launch_win_band_pass(nl, w.row_cnt.p, w.pool_val.p, tau_d, w.passrow.p, nullptr, st, base.half,
                               w.pool_col.p, P.row_begin);
          launch_reduce_sum(w.passrow.p, nl, w.partial.p, w.scal.p + 1, st);
          Sp = allsum(P, d2h(w.scal.p + 1, st));
        }
        b = sqrtl((long double)F + (long double)Sp);
        m = b / epsf;
        passes++;
        REQUIRE(passes < 256, SEXPM_EINTERNAL, "Algorithm 4.1 pass cap reached (Theorem 4.1)");
      }
      tau = (double)epsf;
    }
    // nnz(S^_i) = sure keeps + band values above tau
    int64_t kept = hi[1];
    if (eps_g > 0.0 && !(passes == 1 && tau == eps_g) && hi[2] > 0) {
      launch_win_band_pass(nl, w.row_cnt.p, w.pool_val.p, tau, nullptr, w.cnt2.p, st, base.half, w.pool_col.p,
                           P.row_begin);
      launch_reduce_sum_i64(w.cnt2.p, nl, w.i64tmp.p + 6, st);
      kept += d2h(w.i64tmp.p + 6, st);
    }
    const int64_t nnz = (int64_t)allsum(P, (double)kept);
    const int64_t kept_local = kept;
    float kms = 0.f;
    CK(cudaEventElapsedTime(&kms, k0, k1));
    const double hw = W.half ? 0.5 : 1.0;  // the half window moves about half the planes
    const double bytes = 8.0 * hw * (double)nl * (W.lcnt[i - 1] + W.ccnt[i - 2] + W.ccnt[i - 1] + W.lcnt[i]) +
                         12.0 * (double)hi[2] + 40.0 * (double)nl;
    if (i < SEXPM_MAXSTEP) {
      S.taylor_nnz_unf[i] = (int64_t)allsum(P, (double)hi[0]);
      S.taylor_nnz[i] = nnz;
      S.taylor_passes[i] = passes;
      S.taylor_tau[i] = tau;
      S.taylor_numeric_ms[i] = kms;
      S.taylor_numeric_bytes[i] = bytes;
      S.taylor_fmas_i[i] = allsum(P, prods);
      S.taylor_fallback_rows[i] = 0;
    }
    S.taylor_fmas += allsum(P, prods);
    S.taylor_bytes += bytes;
    if (getenv("SEXPM_STEP_LOG"))
      fprintf(stderr, "[sexpm run] taylor %d (window): nnz %lld passes %d kernel %.2f ms (%.0f GB/s) band %lld\n", i,
              (long long)nnz, passes, kms, bytes / (kms * 1e6), (long long)hi[2]);
    if (nnz == 0) {  // S^_i = 0: all later terms vanish
      if (i < SEXPM_MAXSTEP) S.taylor_ms[i] = step_ms();
      t0_complete = true;  // this launch already added S^_{i-1}: T^_0 is final
      break;
    }
    M_eff = i;
    tau_prev = tau;
    prev_nnz_local = kept_local;
    sa ^= 1;
    if (i < SEXPM_MAXSTEP) S.taylor_ms[i] = step_ms();
  }
  // T^_0 = T^_0^(m-1) + S^_m as CSR: count, scan, write
  const auto h_fin = std::chrono::steady_clock::now();
  {
    const int m = M_eff;
    WinArgs a = base;
    a.prev_is_h0 = m == 1;
    a.pS = ck_s[sa]->p;
    a.tau_prev = tau_prev;
    a.T0old = t0buf.p;
    a.c1cnt = W.ccnt[m];
    a.mapC = W.mapC.p + W.coff[m];
    a.mapW = W.mapW.p + W.coff[m];
    if (t0_complete) {  // T^_0 = the buffer over cum_m as it stands
      a.mapC = W.cumU.p + W.coff[m];
      a.mapW = W.neg1.p;
    }
    a.coffs = W.coffs.p + W.coff[m];
    a.sym = P.sym_sq ? 1 : 0;  // T^_0 exactly symmetric for the symmetric squarings (R21)
    launch_taylor_win_final(a, w.cnt.p, nullptr, nullptr, nullptr, st);
    T.nrows = nl;
    T.row0 = P.row_begin;
    T.padded = false;
    T.rp.ensure((size_t)nl + 1, st);
    launch_exclusive_scan(w.cnt.p, nl, T.rp.p, w.scan_tmp.p, st);
    T.nnz = d2h(T.rp.p + nl, st);
    T.col.ensure((size_t)std::max<int64_t>(T.nnz, 1), st);
    T.val.ensure((size_t)std::max<int64_t>(T.nnz, 1), st);
    launch_taylor_win_final(a, nullptr, T.rp.p, T.col.p, T.val.p, st);
    CK(cudaGetLastError());
    S.taylor_bytes += 16.0 * (double)nl * a.c1cnt * 2 + 12.0 * (double)T.nnz;
    if (getenv("SEXPM_STEP_LOG")) {
      CK(cudaStreamSynchronize(st));
      fprintf(stderr, "[sexpm run] taylor (window): setup %.1f ms, T^_0 to CSR %.1f ms (host wall)\n",
              std::chrono::duration<double, std::milli>(h_loop - h_start).count(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h_fin).count());
    }
  }
  cudaEventDestroy(k0);
  cudaEventDestroy(k1);
  // the checkpoints live for the Taylor phase only
  return M_eff;
}

static void do_run(sexpm_plan_s &P) {
  cudaStream_t st = P.st;
  sexpm_stats &S = P.stats;
  const long long launches0 = g_kernel_launches;
  memset(&S, 0, sizeof(S));
  S.struct_size = sizeof(sexpm_stats);
  S.M = P.M;
  S.N = P.N;
  S.normal = P.normal;
  S.world = P.world;
  S.rank = P.rank;
  S.norm = P.norm;
  S.a = P.a;
  S.r0 = (double)P.r0;
  S.eps_g0 = P.eps_g0;
  S.ms_plan = P.plan_ms;
  cudaEvent_t ev_start, ev_taylor, ev_sq, ev_end, a0, a1;
  CK(cudaEventCreate(&ev_start));
  CK(cudaEventCreate(&ev_taylor));
  CK(cudaEventCreate(&ev_sq));
  CK(cudaEventCreate(&ev_end));
  CK(cudaEventCreate(&a0));
  CK(cudaEventCreate(&a1));
  auto step_ms = [&]() {
    CK(cudaEventRecord(a1, st));
    CK(cudaEventSynchronize(a1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a0, a1));
    return (double)ms;
  };
  CK(cudaEventRecord(ev_start, st));
  // the first Taylor term tries the short-row kernel K5s only if S^_2 = H0 H0 / 2 can fit
  // its window: a row of H0 H0 spans at most 2 (dmax - dmin) + 1 columns
  P.dia_short_ok = 2 * ((int64_t)P.dia_dmax - P.dia_dmin) + 1 <= 64;
  P.taylor_block = false;
  const int64_t nl = P.row_end - P.row_begin;
  // symmetric squarings (option sym_squaring, reading R21): H bit-exactly symmetric, one GPU,
  // the tensor-core block kernel
  P.sym_sq = sym_path_enabled(P);
  DCsr &H0loc = P.H0loc;
  DCsr &T = P.T, &Tn = P.Tn, &Sc = P.S, &Sn = P.Sn;
  // ---- Taylor phase ----
  int M_eff = 0;
  if (P.M >= 1 && P.win.ok) {
    M_eff = taylor_window(P, T, step_ms, a0);
    S.taylor_window = 1;
  } else if (P.M == 0) {  // reading R9: T^_0 = 0
    T.nrows = nl;
    T.row0 = P.row_begin;
    T.nnz = 0;
    T.padded = false;
    T.rp.ensure((size_t)nl + 1, st);
    CK(cudaMemsetAsync(T.rp.p, 0, (nl + 1) * sizeof(int64_t), st));
    T.col.ensure(1, st);
    T.val.ensure(1, st);
  } else {
    copy_csr(P, H0loc.view(), T);  // T^_0^(1) = S_1 = H0
    copy_csr(P, H0loc.view(), Sc);
    M_eff = 1;
    for (int i = 2; i <= P.M; i++) {
      CK(cudaEventRecord(a0, st));
      StepReport rep;
      filtered_product(P, Sc.view(), P.H0full.view(), 0.0, (double)i, P.eps_g0, Sn, rep, &P.H0T,
                       false, &T, &Tn);  // S^_i and T^_0^(i) = T^_0^(i-1) + S^_i
      if (i < SEXPM_MAXSTEP) {
        S.taylor_nnz_unf[i] = rep.nnz_unf;
        S.taylor_nnz[i] = rep.nnz;
        S.taylor_passes[i] = rep.passes;
        S.taylor_tau[i] = rep.tau;
        S.taylor_numeric_ms[i] = rep.numeric_ms;
        S.taylor_numeric_bytes[i] = rep.numeric_bytes;
        S.taylor_fmas_i[i] = rep.fmas;
        S.taylor_fallback_rows[i] = rep.window_rows;
      }
      S.taylor_fmas += rep.fmas;
      S.taylor_bytes += 12.0 * (double)Sc.nnz + 12.0 * (double)Sn.nnz + 16.0 * (double)nl;
      if (rep.nnz == 0) {  // S^_i = 0: all later terms vanish
        if (i < SEXPM_MAXSTEP) S.taylor_ms[i] = step_ms();
        break;
      }
      M_eff = i;
      S.taylor_bytes += 12.0 * ((double)T.nnz + (double)Tn.nnz);
      swap_csr(T, Tn);
      swap_csr(Sc, Sn);
      if (i < SEXPM_MAXSTEP) S.taylor_ms[i] = step_ms();
      if (getenv("SEXPM_STEP_LOG"))
        fprintf(stderr, "[sexpm run] taylor %d: nnz %lld passes %d numeric %.1f ms fallback %lld\n", i,
                (long long)rep.nnz, rep.passes, rep.numeric_ms, (long long)rep.window_rows);
    }
  }
  P.M_eff = M_eff;
  S.M_eff = M_eff;
  if (T.padded) {  // T^_0 to plain CSR (one pass; the merges wrote it with row capacities)
    Workspace &w = P.ws;
    const size_t nl1 = (size_t)std::max<int64_t>(nl, 1);
    w.cnt.ensure(nl1, st);
    w.scan_tmp.ensure((size_t)scan_tmp_elems(nl) + 1, st);
    w.rs.ensure(nl1, st);
    w.l1r.ensure(nl1, st);
    w.l2r.ensure(nl1, st);
    Tn.nrows = nl;
    Tn.row0 = T.row0;
    Tn.rp.ensure((size_t)nl + 1, st);
    launch_exclusive_scan(T.len.p, nl, Tn.rp.p, w.scan_tmp.p, st);
    Tn.nnz = d2h(Tn.rp.p + nl, st);
    Tn.col.ensure((size_t)std::max<int64_t>(Tn.nnz, 1), st);
    Tn.val.ensure((size_t)std::max<int64_t>(Tn.nnz, 1), st);
    Tn.padded = false;
    // tau = 0 keeps every entry (the merges never write zeros)
    launch_compact_write(nl, T.row0, T.rp.p, T.len.p, T.col.p, T.val.p, 0.0, Tn.rp.p, Tn.col.p,
                         Tn.val.p, w.rs.p, w.l1r.p, w.l2r.p, st);
    swap_csr(T, Tn);
  }
  // symmetric squarings need T^_0 exactly symmetric: the window path wrote it so; otherwise
  // keep (r, c) iff (c, r) is present, both with the upper triangle's value (R21)
  if (P.sym_sq && M_eff >= 2 && !S.taylor_window) {
    Workspace &w = P.ws;
    w.cnt.ensure((size_t)std::max<int64_t>(nl, 1), st);
    w.scan_tmp.ensure((size_t)scan_tmp_elems(nl) + 1, st);
    launch_sym_intersect(T.view(), w.cnt.p, nullptr, nullptr, nullptr, st);
    Tn.nrows = nl;
    Tn.row0 = T.row0;
    Tn.padded = false;
    Tn.rp.ensure((size_t)nl + 1, st);
    launch_exclusive_scan(w.cnt.p, nl, Tn.rp.p, w.scan_tmp.p, st);
    Tn.nnz = d2h(Tn.rp.p + nl, st);
    Tn.col.ensure((size_t)std::max<int64_t>(Tn.nnz, 1), st);
    Tn.val.ensure((size_t)std::max<int64_t>(Tn.nnz, 1), st);
    launch_sym_intersect(T.view(), nullptr, Tn.rp.p, Tn.col.p, Tn.val.p, st);
    swap_csr(T, Tn);
  }
  CK(cudaEventRecord(ev_taylor, st));
  // squarings in aggregate order (option sq_order, one GPU): T^_0 relabelled once here, E
  // mapped back after the last squaring (the SSAT baseline keeps the index order: its
  // products must match the oracle's bit for bit)
  P.sq_tiled = false;
  if (P.o.sq_order == 1 && P.N >= 1 && !P.o.ssat && P.M >= 1) {
    wait_order(P);
    if (P.tperm_ready) {
      if (P.sym_sq && P.world == 1 && !getenv("SEXPM_NO_FUSED_RELABEL")) {
        P.t_index_pending = true;  // the first squaring's BSR build relabels (no CSR pass)
      } else {
        permute_csr(P, T.view(), P.tperm_loc.p, P.tinv.p, Tn);  // row i <- row tperm[i], col c -> tinv[c]
        swap_csr(T, Tn);
      }
      P.sq_tiled = true;
      S.sq_order_used = P.agg_kind;
    }
  }
  // stats of T^_0
  {
    Workspace &w = P.ws;
    w.rs.ensure((size_t)std::max<int64_t>(nl, 1), st);
    w.l1r.ensure((size_t)std::max<int64_t>(nl, 1), st);
    w.l2r.ensure((size_t)std::max<int64_t>(nl, 1), st);
    w.partial.ensure(1024, st);
    w.scal.ensure(8, st);
    w.i64tmp.ensure(8, st);
    launch_row_stats(T.view(), w.rs.p, w.l1r.p, w.l2r.p, st);
    launch_reduce_sum(w.rs.p, nl, w.partial.p, w.scal.p, st);
    launch_reduce_max_i64(w.l1r.p, nl, w.i64tmp.p + 0, st);
    launch_reduce_max_i64(w.l2r.p, nl, w.i64tmp.p + 1, st);
    S.sq_normIT[0] = sqrt(allsum(P, d2h(w.scal.p, st)));
    S.sq_l1[0] = (int64_t)allmax(P, (double)d2h(w.i64tmp.p + 0, st));
    S.sq_l2[0] = (int64_t)allmax(P, (double)d2h(w.i64tmp.p + 1, st));
    S.sq_nnz[0] = (int64_t)allsum(P, (double)T.nnz);
  }
  // ---- squarings ----
  const bool ssat = P.o.ssat != 0;
  if (ssat && P.N >= 1) {  // SSAT baseline: E_0 = I + T^_0, then E_i = E_{i-1}^2 (no filter)
    DCsr &I = P.Ibuf;
    I.nrows = nl;
    I.row0 = P.row_begin;
    I.nnz = nl;
    I.rp.ensure((size_t)nl + 1, st);
    I.col.ensure((size_t)std::max<int64_t>(nl, 1), st);
    I.val.ensure((size_t)std::max<int64_t>(nl, 1), st);
    launch_identity(nl, P.row_begin, I.rp.p, I.col.p, I.val.p, st);
    merge_add(P, T.view(), I.view(), Tn);
    swap_csr(T, Tn);
  }
  long double ri = P.r0;
  double normIT = S.sq_normIT[0];
  int64_t l1 = S.sq_l1[0], l2 = S.sq_l2[0];
  for (int i = 1; i <= P.N; i++) {
    CK(cudaEventRecord(a0, st));
    ri = 2.0L * ri;  // r_i = 2 r_{i-1}
    double eps_g = P.o.threshold_mode == 1 ? (double)((long double)P.a * ri)
                                           : (double)((long double)P.a * ri * (long double)normIT);
    if (!P.o.filter || ssat) eps_g = 0.0;
    StepReport rep;
    // last squaring: E = I + T^_N is written by its compaction, no separate merge
    const bool fuse_I = (i == P.N) && !P.o.output_T && !ssat;
    DCsr &dst = fuse_I ? P.E : Tn;
    const double self = ssat ? 0.0 : 2.0;  // T~ = 2T + T^2 (Eq. 4.15), or E^2 (SSAT)
    const int64_t nnz_in = P.blk_valid ? P.blk_nnz : T.nnz;
    P.sq_index = i;
    if (P.world == 1) {
      // the symmetric path hands the iterate on in block form up to the last squaring
      P.blk_out = P.sym_sq && i < P.N && !ssat && !getenv("SEXPM_NO_BLOCK_ITER");
      CsrView Tv = T.view();
      if (P.blk_valid) {  // T^ lives in ws.bsrB: no CSR of it exists
        Tv = CsrView();
        Tv.nrows = nl;
        Tv.row0 = P.row_begin;
        Tv.nnz = P.blk_nnz;
      }
      filtered_product(P, Tv, Tv, self, 1.0, eps_g, dst, rep, nullptr, fuse_I);
      if (rep.relabel_needed || rep.need_csr) {  // back to the CSR path, then the product again
        if (rep.need_csr) {  // T^ from its block view
          Workspace &w = P.ws;
          w.cnt.ensure((size_t)std::max<int64_t>(nl, 1), st);
          w.scan_tmp.ensure((size_t)scan_tmp_elems(nl) + 1, st);
          const BsrView V = w.bsrB.view();
          launch_bsr_to_csr(V, nl, w.cnt.p, nullptr, nullptr, nullptr, st);
          T.nrows = nl;
          T.row0 = P.row_begin;
          T.padded = false;
          T.rp.ensure((size_t)nl + 1, st);
          launch_exclusive_scan(w.cnt.p, nl, T.rp.p, w.scan_tmp.p, st);
          T.nnz = d2h(T.rp.p + nl, st);
          T.col.ensure((size_t)std::max<int64_t>(T.nnz, 1), st);
          T.val.ensure((size_t)std::max<int64_t>(T.nnz, 1), st);
          launch_bsr_to_csr(V, nl, nullptr, T.rp.p, T.col.p, T.val.p, st);
          P.blk_valid = false;
        } else {  // relabel T^_0 after all
          P.t_index_pending = false;
          permute_csr(P, T.view(), P.tperm_loc.p, P.tinv.p, Tn);
          swap_csr(T, Tn);
        }
        P.blk_out = false;
        rep = StepReport();
        filtered_product(P, T.view(), T.view(), self, 1.0, eps_g, dst, rep, nullptr, fuse_I);
      }
      P.t_index_pending = false;
      P.blk_out = false;
    } else {
      const auto x0 = std::chrono::steady_clock::now();
      exchange_halo(P, T, l1, l2, P.Bhalo);
      if (i < SEXPM_MAXSTEP)
        S.sq_exchange_ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - x0).count();
      filtered_product(P, T.view(), P.Bhalo.view(), self, 1.0, eps_g, dst, rep, nullptr, fuse_I);
    }
    const double ms = step_ms();
    if (i < SEXPM_MAXSTEP) {
      S.sq_nnz_unf[i] = rep.nnz_unf;
      S.sq_nnz[i] = rep.nnz;
      S.sq_staged[i] = (int64_t)allsum(P, (double)rep.staged);
      S.sq_passes[i] = rep.passes;
      S.sq_eps_g[i] = eps_g;
      S.sq_tau[i] = rep.tau;
      S.sq_normIT[i] = sqrt(rep.normIT2);
      S.sq_l1[i] = rep.l1;
      S.sq_l2[i] = rep.l2;
      S.sq_fmas[i] = allsum(P, rep.fmas);
      S.sq_ms[i] = ms;
      S.sq_numeric_ms[i] = rep.numeric_ms;
      S.sq_numeric_bytes[i] = rep.numeric_bytes;
      S.sq_fallback_rows[i] = rep.window_rows;
      S.sq_first_ms[i] = rep.first_ms;
      S.sq_kernel_ms[i] = rep.kernel_ms > 0.f ? rep.kernel_ms : rep.first_ms;
      S.sq_bsr_blocks[i] = rep.bsr_blocks;
      S.sq_block_products[i] = rep.block_products;
      S.sq_assemble_ms[i] = rep.asm_ms;
      S.sq_sym_used += rep.sym ? 1 : 0;
      S.sq_bytes[i] = 12.0 * (double)nnz_in + 12.0 * (double)rep.nnz + 16.0 * (double)nl;
    }
    if (getenv("SEXPM_STEP_LOG"))
      fprintf(stderr, "[sexpm run] squaring %d: nnz %lld passes %d numeric %.1f ms (first kernel %.1f) fallback %lld\n",
              i, (long long)rep.nnz, rep.passes, rep.numeric_ms, rep.first_ms, (long long)rep.window_rows);
    normIT = sqrt(rep.normIT2);
    l1 = rep.l1;
    l2 = rep.l2;
    if (!fuse_I && !P.blk_valid) swap_csr(T, Tn);  // (block form: T^ lives in ws.bsrB)
  }
  P.blk_valid = false;
  CK(cudaEventRecord(ev_sq, st));
  // ---- e^H = I + T^_N ----
  if (ssat && P.N >= 1) {
    copy_csr(P, T.view(), P.E);  // E_N of the SSAT baseline
  } else if (P.N >= 1 && !P.o.output_T) {
    // already written by the last squaring's compaction
  } else if (P.o.output_T) {
    copy_csr(P, T.view(), P.E);
  } else {
    DCsr &I = P.Ibuf;
    I.nrows = nl;
    I.row0 = P.row_begin;
    I.nnz = nl;
    I.rp.ensure((size_t)nl + 1, st);
    I.col.ensure((size_t)std::max<int64_t>(nl, 1), st);
    I.val.ensure((size_t)std::max<int64_t>(nl, 1), st);
    launch_identity(nl, P.row_begin, I.rp.p, I.col.p, I.val.p, st);
    merge_add(P, T.view(), I.view(), P.E);
  }
  if (P.sq_tiled) {  // back to index order: row r <- row tinv[r], col c' -> tperm[c']
    DCsr &spare = (&T == &P.E) ? Tn : (T.nnz >= P.E.nnz ? T : Tn);  // an iterate no longer needed
    permute_csr(P, P.E.view(), P.tinv_loc.p, P.tperm.p, spare);
    swap_csr(P.E, spare);
    P.sq_tiled = false;
  }
  CK(cudaEventRecord(ev_end, st));
  CK(cudaStreamSynchronize(st));
  float t1, t2, t3, t4;
  CK(cudaEventElapsedTime(&t1, ev_start, ev_taylor));
  CK(cudaEventElapsedTime(&t2, ev_taylor, ev_sq));
  CK(cudaEventElapsedTime(&t3, ev_sq, ev_end));
  CK(cudaEventElapsedTime(&t4, ev_start, ev_end));
  S.ms_taylor = t1;
  S.ms_squaring = t2;
  S.ms_finalize = t3;
  S.ms_total = t4;
  S.nnz_out = P.E.nnz;
  S.gpu_launches = (int32_t)(g_kernel_launches - launches0);
  S.retries = P.retries;
  P.retries = 0;
  {
    std::lock_guard<std::mutex> lk(cache::mu);
    S.cache_hits = cache::hits - P.cache0[0];
    S.cache_misses = cache::misses - P.cache0[1];
    S.cache_releases = cache::releases - P.cache0[2];
    S.cache_bytes_cached = cache::bytes_cached;
    S.cache_bytes_allocated = cache::bytes_allocated;
    S.ms_order_host = P.order_host_ms;
    S.ms_order_wait = P.order_wait_ms;
  }
  if (P.o.reorder) {  // N3: E = P^T E' P (row r <- row inv[r], col c' -> perm[c'])
    DCsr &spare = (&P.T == &P.E) ? P.Tn : (P.T.nnz >= P.E.nnz ? P.T : P.Tn);  // free iterates
    permute_csr(P, P.E.view(), P.inv.p, P.perm.p, spare);
    swap_csr(P.E, spare);
    CK(cudaStreamSynchronize(st));
  }
  for (cudaEvent_t e : {ev_start, ev_taylor, ev_sq, ev_end, a0, a1}) cudaEventDestroy(e);
  P.have_result = true;
}

// ------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------
#define ABI_BEGIN try {
#define ABI_END                                                  \
  }                                                              \
  catch (const SxError &e) {                                     \
    g_err = e.msg;                                               \
    return e.code;                                               \
  }                                                              \
  catch (const std::exception &e) {                              \
    g_err = e.what();                                            \
    return SEXPM_EINTERNAL;                                      \
  }                                                              \
  catch (...) {                                                  \
    g_err = "unknown exception";                                 \
    return SEXPM_EINTERNAL;                                      \
  }                                                              \
  return SEXPM_OK;

extern "C" {

const char *sexpm_last_error(void) { return g_err.c_str(); }

int sexpm_kernel_launches(int64_t *count) {
  if (!count) return SEXPM_EINVAL;
  *count = (int64_t)g_kernel_launches;
  return SEXPM_OK;
}

int sexpm_fp64_peak(double *dfma_tflops, double *dmma_tflops) {
  ABI_BEGIN
  REQUIRE(dfma_tflops || dmma_tflops, SEXPM_EINVAL, "bad args");
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double *out = nullptr;
  CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * sizeof(double)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int which = 0; which < 2; which++) {
    double *dst = which == 0 ? dfma_tflops : dmma_tflops;
    if (!dst) continue;
    launch_fp64_peak(which, sms, out, st);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {  // best of 5, CUDA events on the launching stream
      CK(cudaEventRecord(e0, st));
      launch_fp64_peak(which, sms, out, st);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    *dst = fp64_peak_flops_per_launch(which, sms) / (best * 1e-3) / 1e12;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(cudaFree(out));
  CK(cudaStreamDestroy(st));
  ABI_END
}

int sexpm_abi_sizes(uint32_t *sizes) {
  if (!sizes) return SEXPM_EINVAL;
  sizes[0] = sizeof(sexpm_options);
  sizes[1] = sizeof(sexpm_stats);
  sizes[2] = sizeof(sexpm_csr_in);
  sizes[3] = sizeof(sexpm_csr_out);
  return SEXPM_OK;
}

int sexpm_options_init(sexpm_options *o) {
  if (!o) return SEXPM_EINVAL;
  memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(sexpm_options);
  o->plan_norm = 0;
  o->normal = -1;
  o->threshold_mode = 0;
  o->filter = 1;
  o->m_cap = 120;
  o->n_window = 50;
  o->force_M = -1;
  o->force_N = -1;
  o->output_T = 0;
  o->window_cols = 0;
  o->kernel = 0;
  o->ssat = 0;
  o->reorder = 0;
  o->sq_order = 1;
  o->exact_products = 0;
  o->sym_squaring = -1;
  o->e_r = 0.1;
  o->stream = nullptr;
  o->nccl_comm = nullptr;
  return SEXPM_OK;
}

int sexpm_nccl_unique_id(void *id128) {
  ABI_BEGIN
  REQUIRE(id128, SEXPM_EINVAL, "null id");
  ncclUniqueId id;
  NK(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id128, &id, sizeof(id));
  ABI_END
}

int sexpm_nccl_comm_init(int rank, int world, const void *id128, void **comm) {
  ABI_BEGIN
  REQUIRE(id128 && comm && world >= 1 && rank >= 0 && rank < world, SEXPM_EINVAL, "bad args");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t nc;
  NK(nccl().CommInitRank(&nc, world, id, rank));
  SxComm *c = new SxComm();
  c->kind = 0;
  c->world = world;
  c->rank = rank;
  c->nccl = nc;
  *comm = c;
  ABI_END
}

int sexpm_virtual_comm_create(int world, void **comms) {
  ABI_BEGIN
  REQUIRE(comms && world >= 1 && world <= 64, SEXPM_EINVAL, "bad args");
  VirtualHub *hub = new VirtualHub();
  hub->W = world;
  hub->ag.assign((size_t)world, nullptr);
  hub->sent.assign((size_t)world, {});
  hub->refs = world;
  for (int r = 0; r < world; r++) {
    SxComm *c = new SxComm();
    c->kind = 1;
    c->world = world;
    c->rank = r;
    c->hub = hub;
    comms[r] = c;
  }
  ABI_END
}

int sexpm_nccl_comm_destroy(void *comm) {
  ABI_BEGIN
  if (comm) {
    SxComm *c = as_comm(comm);
    if (c->kind == 0) NK(nccl().CommDestroy(c->nccl));
    else if (--c->hub->refs == 0) delete c->hub;
    c->magic = 0;
    delete c;
  }
  ABI_END
}

static sexpm_plan_s *new_plan(const sexpm_options *o) {
  sexpm_plan_s *P = new sexpm_plan_s();
  if (o) {
    REQUIRE(o->struct_size == sizeof(sexpm_options), SEXPM_EINVAL, "sexpm_options ABI mismatch");
    REQUIRE(!(o->ssat && o->output_T), SEXPM_EINVAL, "ssat has no incremental part T to return");
    P->o = *o;
  } else {
    sexpm_options_init(&P->o);
  }
  CK(cudaGetDevice(&P->dev));
  static std::mutex prop_mu;
  static std::map<int, cudaDeviceProp> props;  // cudaGetDeviceProperties is slow: once per device
  cudaDeviceProp prop;
  {
    std::lock_guard<std::mutex> lk(prop_mu);
    auto it = props.find(P->dev);
    if (it == props.end()) {
      CK(cudaGetDeviceProperties(&prop, P->dev));
      props[P->dev] = prop;
    } else {
      prop = it->second;
    }
  }
  P->sm_count = prop.multiProcessorCount;
  P->smem_per_sm = prop.sharedMemPerMultiprocessor;
  {
    int role = 0;
    for (DCsr *c : {&P->T, &P->Tn, &P->S, &P->Sn, &P->E, &P->Bhalo}) {
      c->rp.role = role++;
      c->col.role = role++;
      c->val.role = role++;
    }
    P->ws.pool_col.role = role++;
    P->ws.pool_val.role = role++;
    for (BsrBufs *b : {&P->ws.bsrB, &P->ws.bsrA}) {
      b->bval.role = role++;
      b->bcol.role = role++;
      b->tk.role = role++;
      b->tk_tmp.role = role++;
      b->tb.role = role++;
      b->tb_tmp.role = role++;
      b->keys_tmp.role = role++;
      b->sort_tmp.role = role++;
    }
    P->ws.bscr.role = role++;
    P->ws.sym_bstore.role = role++;
    P->ws.sym_cj.role = role++;
    REQUIRE(role <= cache::kRoles, SEXPM_EINTERNAL, "device-block cache: too many buffer roles");
  }
  {
    std::lock_guard<std::mutex> lk(cache::mu);
    P->cache0[0] = cache::hits;
    P->cache0[1] = cache::misses;
    P->cache0[2] = cache::releases;
  }
  int window = P->o.window_cols > 0 ? P->o.window_cols : 8192;
  int smem = numeric_smem_bytes(window);
  REQUIRE(smem <= (int)prop.sharedMemPerBlockOptin - 2048, SEXPM_EINVAL, "window too large");
  P->numeric_blocks_per_sm = std::max(1, std::min(4, (int)(prop.sharedMemPerMultiprocessor / (smem + 4096))));
  // CTAs per SM from shared memory: dynamic + static (< 6 KB) + the 1 KB per-CTA reserve
  P->paged_blocks_per_sm = std::max(1, std::min(8, (int)(prop.sharedMemPerMultiprocessor / (paged_smem_bytes() + 7168))));
  if (P->o.stream) {
    P->st = (cudaStream_t)P->o.stream;
  } else {
    CK(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
    P->own_stream = true;
  }
  {  // once per device: the pool keeps freed memory (no trimming at synchronisation points)
    static std::mutex pool_mu;
    static bool pool_set[64] = {};
    std::lock_guard<std::mutex> lk(pool_mu);
    cudaMemPool_t pool;
    if (P->dev >= 0 && P->dev < 64 && !pool_set[P->dev] &&
        cudaDeviceGetDefaultMemPool(&pool, P->dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      pool_set[P->dev] = true;
    }
  }
  if (P->o.nccl_comm) {
    SxComm *c = as_comm(P->o.nccl_comm);
    if (c->kind == 0) {
      auto t = std::make_unique<NcclTransport>();
      t->comm = c->nccl;
      P->tr = std::move(t);
    } else {
      auto t = std::make_unique<VirtualTransport>();
      t->hub = c->hub;
      P->tr = std::move(t);
    }
    P->tr->world = P->world = c->world;
    P->tr->rank = P->rank = c->rank;
  }
  return P;
}

static int plan_common(const sexpm_csr_in *H, double eps_tol, const sexpm_options *o,
                       sexpm_plan_t *out, bool host) {
  if (!out || !H) {
    g_err = "null argument";
    return SEXPM_EINVAL;
  }
  *out = nullptr;
  sexpm_plan_s *P = nullptr;
  try {
    const auto tnp = std::chrono::steady_clock::now();
    P = new_plan(o);
    if (getenv("SEXPM_PLAN_LOG"))
      fprintf(stderr, "[sexpm plan] %-28s %8.2f ms\n", "new_plan",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tnp).count());
    if (host) {
      // copy the host CSR in (H2D inside the call, for end-to-end timing)
      sexpm_csr_in D = *H;
      const int64_t rows = H->row_end - H->row_begin;
      REQUIRE(rows >= 0 && H->rowptr, SEXPM_EINVAL, "bad host CSR");
      DCsr tmp;
      tmp.rp.alloc((size_t)rows + 1, P->st);
      tmp.col.alloc((size_t)std::max<int64_t>(H->nnz, 1), P->st);
      tmp.val.alloc((size_t)std::max<int64_t>(H->nnz, 1), P->st);
      CK(cudaMemcpyAsync(tmp.rp.p, H->rowptr, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, P->st));
      if (H->nnz) {
        CK(cudaMemcpyAsync(tmp.col.p, H->colidx, H->nnz * sizeof(int32_t), cudaMemcpyHostToDevice, P->st));
        CK(cudaMemcpyAsync(tmp.val.p, H->vals, H->nnz * sizeof(double), cudaMemcpyHostToDevice, P->st));
      }
      D.rowptr = tmp.rp.p;
      D.colidx = tmp.col.p;
      D.vals = tmp.val.p;
      do_plan(*P, &D, eps_tol);
    } else {
      do_plan(*P, H, eps_tol);
    }
    *out = P;
    return SEXPM_OK;
  } catch (const SxError &e) {
    g_err = e.msg;
    if (P) {
      if (P->own_stream) cudaStreamSynchronize(P->st);
      delete P;
    }
    return e.code;
  } catch (...) {
    g_err = "unknown exception in sexpm_plan";
    delete P;
    return SEXPM_EINTERNAL;
  }
}

int sexpm_plan(const sexpm_csr_in *H, double eps_tol, const sexpm_options *o, sexpm_plan_t *out) {
  return plan_common(H, eps_tol, o, out, false);
}

int sexpm_plan_host(const sexpm_csr_in *H, double eps_tol, const sexpm_options *o,
                    sexpm_plan_t *out) {
  return plan_common(H, eps_tol, o, out, true);
}

int sexpm_run(sexpm_plan_t p, sexpm_csr_out *E) {
  ABI_BEGIN
  REQUIRE(p, SEXPM_EINVAL, "null plan");
  do_run(*p);
  if (E) {
    E->n = p->n;
    E->row_begin = p->row_begin;
    E->row_end = p->row_end;
    E->nnz = p->E.nnz;
    E->rowptr = p->E.rp.p;
    E->colidx = p->E.col.p;
    E->vals = p->E.val.p;
  }
  ABI_END
}

int sexpm_result_copy(sexpm_plan_t p, int64_t *rowptr, int32_t *colidx, double *vals) {
  ABI_BEGIN
  REQUIRE(p && p->have_result, SEXPM_ESTATE, "no result: call sexpm_run first");
  REQUIRE(rowptr && (p->E.nnz == 0 || (colidx && vals)), SEXPM_EINVAL, "null host arrays");
  CK(cudaMemcpyAsync(rowptr, p->E.rp.p, (p->E.nrows + 1) * sizeof(int64_t), cudaMemcpyDefault, p->st));
  if (p->E.nnz) {
    CK(cudaMemcpyAsync(colidx, p->E.col.p, p->E.nnz * sizeof(int32_t), cudaMemcpyDefault, p->st));
    CK(cudaMemcpyAsync(vals, p->E.val.p, p->E.nnz * sizeof(double), cudaMemcpyDefault, p->st));
  }
  CK(cudaStreamSynchronize(p->st));
  ABI_END
}

// A result detached from its plan while its copy to the caller's arrays is in flight
// (sexpm_result_copy_async / sexpm_result_wait).
//
// A host thread waits for the plan's stream and then moves the three arrays on the library's
// copy stream.  Destinations a kernel can write (pinned or registered host memory, device
// memory) are written by k_copy_out, a few resident CTAs storing over the link; the copy
// engines are left to the running plan.  Measured at config 5 with the copy engine instead:
// behind one 14.6 GB copy the next plan's first scalar read-back waited for the whole
// transfer (265 ms); in 4 MB chunks, 2 queued at a time, read-backs on the legacy default
// stream got through, but one read-back per array still waited for that array's whole
// transfer (85 + 180 ms inside the Taylor phase), and on created streams every one did: no
// overlap either way (tools/ce_probe*.py).  Pageable destinations take that chunked path.
struct sexpm_copy_s {
  DBuf<int64_t> rp;
  DBuf<int32_t> col;
  DBuf<double> val;
  int dev = 0;
  cudaEvent_t ready = nullptr;  // the plan's stream has produced E
  std::thread th;
  cudaError_t err = cudaSuccess;
  struct Seg {
    char *dst;
    const char *src;
    size_t bytes;
  } seg[3] = {};
};
static size_t env_size(const char *name, size_t dflt) {
  const char *e = getenv(name);
  return e && atoll(e) > 0 ? (size_t)atoll(e) : dflt;
}
static void copy_worker(sexpm_copy_s *c) {
  const size_t chunk = env_size("SEXPM_COPY_CHUNK_KB", 4096) << 10;
  const int depth = (int)std::min<size_t>(env_size("SEXPM_COPY_DEPTH", 2), 8);
  // one copy stream per device for the life of the process (copies of consecutive results
  // queue on it in order)
  static std::mutex cs_mu;
  static cudaStream_t cs_dev[64] = {};
  cudaStream_t cs = nullptr;
  cudaEvent_t ev[8] = {};
  cudaError_t e = cudaSetDevice(c->dev);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(cs_mu);
    if (!cs_dev[c->dev & 63]) {  // highest priority: its few CTAs become resident at once
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      e = cudaStreamCreateWithPriority(&cs_dev[c->dev & 63], cudaStreamNonBlocking, hi);
    }
    cs = cs_dev[c->dev & 63];
  }
  for (int k = 0; k < depth && e == cudaSuccess; k++)
    e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventSynchronize(c->ready);
  long long q = 0;
  // config 5 (14.6 GB over PCIe 5 x16): 4 CTAs fall short of the link (the next e^H waits 25 ms
  // for the copy), 6 keep up with it (~50 GB/s) and slow the running e^H by 35 ms, 32 by 115 ms
  const int ctas = (int)env_size("SEXPM_COPY_CTAS", 6);
  for (int sgi = 0; sgi < 3 && e == cudaSuccess; sgi++) {
    const sexpm_copy_s::Seg &sg = c->seg[sgi];
    // destinations a kernel can write (pinned / registered host memory, device memory): one
    // kernel of a few resident CTAs per array; pageable host memory: the copy engine
    cudaPointerAttributes pa;
    const bool sm_path = !getenv("SEXPM_COPY_ENGINE") && sg.bytes > 0 &&
                         cudaPointerGetAttributes(&pa, sg.dst) == cudaSuccess &&
                         pa.type != cudaMemoryTypeUnregistered && pa.devicePointer != nullptr;
    cudaGetLastError();
    if (sm_path && launch_copy_out(pa.devicePointer, sg.src, sg.bytes, ctas, cs)) {
      e = cudaGetLastError();
      continue;
    }
    for (size_t o = 0; o < sg.bytes && e == cudaSuccess; o += chunk, q++) {
      if (q >= depth) e = cudaEventSynchronize(ev[q % depth]);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(sg.dst + o, sg.src + o, std::min(chunk, sg.bytes - o), cudaMemcpyDefault, cs);
      if (e == cudaSuccess) e = cudaEventRecord(ev[q % depth], cs);
    }
  }
  if (cs) {
    cudaError_t e2 = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = e2;
  }
  for (int k = 0; k < depth; k++)
    if (ev[k]) cudaEventDestroy(ev[k]);
  c->err = e;
}

int sexpm_result_copy_async(sexpm_plan_t p, int64_t *rowptr, int32_t *colidx, double *vals,
                            sexpm_copy_t *ticket) {
  ABI_BEGIN
  REQUIRE(ticket, SEXPM_EINVAL, "null ticket");
  *ticket = nullptr;
  REQUIRE(p && p->have_result, SEXPM_ESTATE, "no result: call sexpm_run first");
  REQUIRE(rowptr && (p->E.nnz == 0 || (colidx && vals)), SEXPM_EINVAL, "null host arrays");
  sexpm_plan_s &P = *p;
  std::unique_ptr<sexpm_copy_s> c(new sexpm_copy_s());
  c->dev = P.dev;
  CK(cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(c->ready, P.st);
  if (e != cudaSuccess) {
    cudaEventDestroy(c->ready);
    CK(e);
  }
  const int64_t nrows = P.E.nrows, nnz = P.E.nnz;
  // detach E: the copy reads it after the plan is gone; its blocks keep their cache roles, so
  // sexpm_result_wait parks them for the next plan's result
  const int r_rp = P.E.rp.role, r_col = P.E.col.role, r_val = P.E.val.role;
  c->rp = std::move(P.E.rp);
  c->col = std::move(P.E.col);
  c->val = std::move(P.E.val);
  c->rp.role = r_rp;
  c->col.role = r_col;
  c->val.role = r_val;
  P.E.nnz = 0;
  P.have_result = false;
  c->seg[0] = {(char *)rowptr, (const char *)c->rp.p, (size_t)(nrows + 1) * sizeof(int64_t)};
  c->seg[1] = {(char *)colidx, (const char *)c->col.p, (size_t)nnz * sizeof(int32_t)};
  c->seg[2] = {(char *)vals, (const char *)c->val.p, (size_t)nnz * sizeof(double)};
  c->th = std::thread(copy_worker, c.get());
  *ticket = c.release();
  ABI_END
}

int sexpm_result_wait(sexpm_copy_t t) {
  ABI_BEGIN
  if (!t) return SEXPM_OK;
  std::unique_ptr<sexpm_copy_s> c(t);
  if (c->th.joinable()) c->th.join();  // the worker has synchronised its stream
  if (c->ready) cudaEventDestroy(c->ready);
  const cudaError_t e = c->err;
  if (e != cudaSuccess) cudaDeviceSynchronize();  // nothing may still read the blocks
  cache::freeing_idle = true;  // the copy is complete: E's blocks are idle, park them
  c.reset();
  cache::freeing_idle = false;
  CK(e);
  ABI_END
}

int sexpm_apply(sexpm_plan_t p, int64_t m, const double *X, int64_t ldx, double *Y, int64_t ldy,
                int32_t steps) {
  ABI_BEGIN
  REQUIRE(p, SEXPM_EINVAL, "null plan");
  REQUIRE(p->have_result, SEXPM_ESTATE, "no result: call sexpm_run first");
  REQUIRE(m >= 0 && steps >= 1 && ldx >= m && ldy >= m, SEXPM_EINVAL, "bad m / ld / steps");
  REQUIRE(m == 0 || (X && Y), SEXPM_EINVAL, "null X or Y");
  sexpm_plan_s &P = *p;
  const int64_t n = P.E.nrows;  // this rank's rows
  REQUIRE(m == 0 || X + (n - 1) * ldx + m <= Y || Y + (n - 1) * ldy + m <= X, SEXPM_EINVAL,
          "X and Y overlap");
  if (P.world == 1 && (m == 0 || n == 0)) return SEXPM_OK;
  const CsrView Ev = P.E.view();
  cudaStream_t st = P.st;
  if (P.world == 1) {
    const double *src = X;
    int64_t lds = ldx;
    for (int s = 1; s <= steps; s++) {
      double *dst = Y;
      int64_t ldd = ldy;
      if (s < steps) {
        DBuf<double> &b = P.apply_buf[s & 1];
        b.ensure((size_t)n * (size_t)m, st);
        dst = b.p;
        ldd = m;
      }
      launch_spmm(Ev, m, src, lds, dst, ldd, st);
      CK(cudaGetLastError());
      src = dst;
      lds = ldd;
    }
    CK(cudaStreamSynchronize(st));
    return SEXPM_OK;
  }
  // several ranks (collective): E's rows of this rank reach the columns [r0 - l2, r1 + l1) of
  // X (Lemma 3.1 with E's bandwidth, measured here); every step assembles those rows of the
  // current block -- own rows copied, the others received from the peers that own them -- and
  // multiplies (global column indices address the assembled block shifted by its first row)
  const int W = P.world, R = P.rank;
  const int64_t r0 = P.row_begin, r1 = P.row_end;
  Workspace &w = P.ws;
  w.rs.ensure((size_t)std::max<int64_t>(n, 1), st);
  w.l1r.ensure((size_t)std::max<int64_t>(n, 1), st);
  w.l2r.ensure((size_t)std::max<int64_t>(n, 1), st);
  w.i64tmp.ensure(8, st);
  int64_t bw[2] = {0, 0};
  if (n) {
    launch_row_stats(Ev, w.rs.p, w.l1r.p, w.l2r.p, st);
    launch_reduce_max_i64(w.l1r.p, n, w.i64tmp.p + 0, st);
    launch_reduce_max_i64(w.l2r.p, n, w.i64tmp.p + 1, st);
    CK(cudaMemcpyAsync(bw, w.i64tmp.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  const int64_t l1 = (int64_t)allmax(P, (double)bw[0]), l2 = (int64_t)allmax(P, (double)bw[1]);
  int64_t need_lo, need_hi;
  halo_need(P.bounds.data(), R, P.n, l1, l2, need_lo, need_hi);
  std::vector<int64_t> rlo(W), rhi(W), slo(W), shi(W);
  halo_ranges_host(W, R, P.bounds.data(), P.n, l1, l2, rlo.data(), rhi.data());
  for (int h = 0; h < W; h++) {
    std::vector<int64_t> lo(W), hi(W);
    halo_ranges_host(W, h, P.bounds.data(), P.n, l1, l2, lo.data(), hi.data());
    slo[h] = lo[R];
    shi[h] = hi[R];
  }
  const size_t rowb = (size_t)m * sizeof(double);
  DBuf<double> xh, xc;  // the assembled rows [need_lo, need_hi) and my rows, both ld = m
  xh.alloc((size_t)std::max<int64_t>(need_hi - need_lo, 1) * (size_t)std::max<int64_t>(m, 1), st);
  xc.alloc((size_t)std::max<int64_t>(n, 1) * (size_t)std::max<int64_t>(m, 1), st);
  const double *src = X;
  int64_t lds = ldx;
  for (int s = 1; s <= steps; s++) {
    if (m && n) {
      CK(cudaMemcpy2DAsync(xc.p, rowb, src, (size_t)lds * sizeof(double), rowb, (size_t)n,
                           cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(xh.p + (size_t)(r0 - need_lo) * m, xc.p, (size_t)n * rowb,
                         cudaMemcpyDeviceToDevice, st));
    }
    std::vector<Transport::Xfer> sends, recvs;
    for (int h = 0; h < W; h++) {
      if (h == R) continue;
      if (shi[h] > slo[h])
        sends.push_back({h, xc.p + (size_t)(slo[h] - r0) * m, nullptr, (size_t)(shi[h] - slo[h]) * rowb});
      if (rhi[h] > rlo[h])
        recvs.push_back({h, nullptr, xh.p + (size_t)(rlo[h] - need_lo) * m, (size_t)(rhi[h] - rlo[h]) * rowb});
    }
    P.tr->exchange(sends, recvs, st);
    double *dst = Y;
    int64_t ldd = ldy;
    if (s < steps) {
      DBuf<double> &b = P.apply_buf[s & 1];
      b.ensure((size_t)std::max<int64_t>(n, 1) * (size_t)std::max<int64_t>(m, 1), st);
      dst = b.p;
      ldd = m;
    }
    // X addressed by global column c at xh + (c - need_lo) m
    if (m && n) launch_spmm(Ev, m, xh.p - (ptrdiff_t)need_lo * m, m, dst, ldd, st);
    CK(cudaGetLastError());
    src = dst;
    lds = ldd;
  }
  CK(cudaStreamSynchronize(st));
  ABI_END
}

int sexpm_rcm(sexpm_plan_t p, const sexpm_csr_in *A, int64_t *perm) {
  ABI_BEGIN
  REQUIRE(p && A && perm, SEXPM_EINVAL, "null argument");
  REQUIRE(A->row_begin == 0 && A->row_end == A->n, SEXPM_EINVAL, "sexpm_rcm needs all rows");
  const CsrView Av = view_of(A);
  DBuf<int64_t> pm, iv;
  compute_rcm(*p, Av, pm, iv);
  if (A->n) CK(cudaMemcpyAsync(perm, pm.p, A->n * sizeof(int64_t), cudaMemcpyDefault, p->st));
  CK(cudaStreamSynchronize(p->st));
  ABI_END
}

int sexpm_spmm(sexpm_plan_t p, const sexpm_csr_in *A, int64_t m, const double *X, int64_t ldx,
               double *Y, int64_t ldy) {
  ABI_BEGIN
  REQUIRE(p && A, SEXPM_EINVAL, "null argument");
  REQUIRE(m >= 0 && ldx >= m && ldy >= m, SEXPM_EINVAL, "bad m / ld");
  REQUIRE(m == 0 || (X && Y), SEXPM_EINVAL, "null X or Y");
  const CsrView Av = view_of(A);
  launch_spmm(Av, m, X, ldx, Y, ldy, p->st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(p->st));
  ABI_END
}

int sexpm_stats_get(sexpm_plan_t p, sexpm_stats *s) {
  ABI_BEGIN
  REQUIRE(p && s, SEXPM_EINVAL, "null argument");
  REQUIRE(s->struct_size == sizeof(sexpm_stats), SEXPM_EINVAL, "sexpm_stats ABI mismatch");
  if (!p->have_result || p->stats.struct_size != sizeof(sexpm_stats)) {
    memset(s, 0, sizeof(*s));
    s->struct_size = sizeof(sexpm_stats);
    s->M = p->M;
    s->N = p->N;
    s->normal = p->normal;
    s->norm = p->norm;
    s->a = p->a;
    s->r0 = (double)p->r0;
    s->eps_g0 = p->eps_g0;
    s->ms_plan = p->plan_ms;
    s->world = p->world;
    s->rank = p->rank;
  } else {
    *s = p->stats;
  }
  ABI_END
}

int sexpm_destroy(sexpm_plan_t p) {
  ABI_BEGIN
  if (!p) return SEXPM_OK;
  cudaStreamSynchronize(p->st);
  cudaStream_t st = p->st;
  bool own = p->own_stream;
  cache::freeing_idle = true;  // the stream is drained: the plan's blocks are idle
  delete p;
  cache::freeing_idle = false;
  cache::mark_idle(st);
  if (own) cudaStreamDestroy(st);
  ABI_END
}

int sexpm_release_cache(void) {
  ABI_BEGIN
  cudaDeviceSynchronize();
  cache::release_all();
  ABI_END
}

int sexpm_filtered_product(sexpm_plan_t p, const sexpm_csr_in *A, const sexpm_csr_in *B,
                           double self_coef, double divisor, double eps_g, sexpm_csr_out *C,
                           int32_t *passes, double *tau, int64_t *nnz_unf) {
  ABI_BEGIN
  REQUIRE(p && A && B && C, SEXPM_EINVAL, "null argument");
  REQUIRE(p->world == 1, SEXPM_EINVAL, "component entry points are single-GPU");
  REQUIRE(divisor != 0.0 && isfinite(eps_g) && eps_g >= 0.0, SEXPM_EINVAL, "bad scalars");
  CsrView Av = view_of(A), Bv = view_of(B);
  p->n = A->n;  // the column dimension (the context plan's own n is that of its 1x1 matrix)
  StepReport rep;
  DCsr out;
  DCsr BT;
  const bool want_pull = self_coef == 0.0 && (p->o.kernel == 0 || p->o.kernel == 6);
  if (want_pull) build_transpose(*p, Bv, A->n, BT);
  filtered_product(*p, Av, Bv, self_coef, divisor, eps_g, out, rep, want_pull ? &BT : nullptr);
  p->E = std::move(out);
  p->have_result = true;  // sexpm_result_copy reads it; sexpm_stats_get is not updated
  C->n = A->n;
  C->row_begin = A->row_begin;
  C->row_end = A->row_end;
  C->nnz = p->E.nnz;
  C->rowptr = p->E.rp.p;
  C->colidx = p->E.col.p;
  C->vals = p->E.val.p;
  if (passes) *passes = rep.passes;
  if (tau) *tau = rep.tau;
  if (nnz_unf) *nnz_unf = rep.nnz_unf;
  ABI_END
}

int sexpm_alg41(sexpm_plan_t p, const double *x, int64_t cnt, double eps_g, double e_r,
                int32_t *passes, double *tau, double *dropped) {
  ABI_BEGIN
  REQUIRE(p && (x || cnt == 0) && cnt >= 0 && e_r > 0.0 && eps_g >= 0.0, SEXPM_EINVAL, "bad args");
  Workspace &w = p->ws;
  w.partial.ensure(1024, p->st);
  w.scal.ensure(8, p->st);
  int np = 0;
  double t = 0.0;
  if (eps_g == 0.0) {
    t = 0.0;
  } else {
    long double m = 1.0L, b = INFINITY, epsf = INFINITY;  // reading R1: first pass always runs
    const long double eg = eps_g, lim = eg * (1.0L + (long double)e_r);
    while (np == 0 || b > lim) {
      epsf = eg / m;
      launch_alg41_pass(x, cnt, (double)epsf, w.partial.p, w.scal.p, p->st);
      double S = d2h(w.scal.p, p->st);
      b = sqrtl((long double)S);
      m = b / epsf;
      np++;
      REQUIRE(np < 256, SEXPM_EINTERNAL, "Algorithm 4.1 pass cap");
    }
    t = (double)epsf;
  }
  // dropped norm: everything <= t
  launch_alg41_pass(x, cnt, t, w.partial.p, w.scal.p, p->st);
  double d = sqrt(d2h(w.scal.p, p->st));
  if (eps_g == 0.0) d = 0.0;
  if (passes) *passes = np;
  if (tau) *tau = t;
  if (dropped) *dropped = d;
  ABI_END
}

int sexpm_plan_scalars(double norm, int normal, double eps_tol, int m_cap, int n_window,
                       int32_t *M, int32_t *N, double *a, double *r0, double *eps_g0) {
  ABI_BEGIN
  REQUIRE(M && N && norm >= 0.0 && std::isfinite(norm) && m_cap >= 0 && n_window >= 0 &&
              (normal == 0 || normal == 1),
          SEXPM_EINVAL, "bad args");
  REQUIRE(eps_tol >= 1e-16 && std::isfinite(eps_tol), SEXPM_ETOL, "eps_tol must be >= 1e-16 (R13)");
  int m = 0, nn = 0;
  REQUIRE(select_MN(norm, eps_tol, m_cap, n_window, m, nn), SEXPM_EINFEASIBLE,
          "Eq. (4.20) infeasible within m_cap / n_window");
  double av = 0.0, e0 = 0.0;
  long double r = 0.0L;
  filter_budgets(norm, normal, m, nn, av, r, e0);
  *M = m;
  *N = nn;
  if (a) *a = av;
  if (r0) *r0 = (double)r;
  if (eps_g0) *eps_g0 = e0;
  ABI_END
}

int sexpm_halo_ranges(int world, int rank, const int64_t *bounds, int64_t n, int64_t l1,
                      int64_t l2, int64_t *recv_lo, int64_t *recv_hi) {
  ABI_BEGIN
  REQUIRE(world >= 1 && rank >= 0 && rank < world && bounds && recv_lo && recv_hi && l1 >= 0 &&
              l2 >= 0,
          SEXPM_EINVAL, "bad args");
  for (int g = 0; g < world; g++)
    REQUIRE(bounds[g] <= bounds[g + 1], SEXPM_EINVAL, "bounds must be non-decreasing");
  REQUIRE(bounds[0] == 0 && bounds[world] == n, SEXPM_EINVAL, "bounds must cover [0, n)");
  halo_ranges_host(world, rank, bounds, n, l1, l2, recv_lo, recv_hi);
  ABI_END
}

int sexpm_partition_rows(int64_t n, const double *work, int world, int64_t *bounds) {
  ABI_BEGIN
  REQUIRE(n >= 0 && world >= 1 && bounds, SEXPM_EINVAL, "bad args");
  double total = 0.0;
  if (work)
    for (int64_t i = 0; i < n; i++) total += work[i];
  else
    total = (double)n;
  bounds[0] = 0;
  double acc = 0.0;
  int g = 1;
  for (int64_t i = 0; i < n && g < world; i++) {
    acc += work ? work[i] : 1.0;
    while (g < world && acc >= total * (double)g / (double)world) {
      bounds[g++] = i + 1;
    }
  }
  while (g < world) bounds[g++] = n;
  bounds[world] = n;
  // interior bounds on multiples of 8: each rank's rows are whole 8-row blocks (K3b)
  for (int k = 1; k < world; k++) bounds[k] = std::min<int64_t>(n, ((bounds[k] + 4) >> 3) << 3);
  for (int k = 1; k <= world; k++)
    if (bounds[k] < bounds[k - 1]) bounds[k] = bounds[k - 1];
  ABI_END
}

}  // extern "C"
