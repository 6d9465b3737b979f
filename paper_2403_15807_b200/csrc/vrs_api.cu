// vrs_api.cu -- libvrs host engine and C ABI (include/vrs.h).
//
// Validation, the predicate's device form, per-call scratch (stream-ordered
// allocator), path dispatch and stream ordering.  Every compute step runs in
// the CUDA kernels of select.cu / scan.cu / gemm_tc.cu / finalize.cu; there is
// no host or CPU fallback for any of them (a device that is not sm_100 gets
// VRS_EUNSUPPORTED).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "vrs_kernels.cuh"


using namespace vrs;

struct vrs_index {
  const float *X;
  int64_t n;
  int32_t d;
  int32_t n_attrs;
  vrs_attr attrs[64];
  int64_t row_offset;
  vrs_allocator alloc;
  int32_t has_alloc;
  float *nx2;
  float *inv_nx;
  int32_t has_zero_row;
  float xmax;              // max row norm (rounded up; the key error bounds)
  void *xb;               // 16-bit shadow corpus [n x d] for the tensor-core selection pass, or nullptr
  int32_t prec16 = 0;     // VRS_PREC_FP16 / VRS_PREC_BF16: the shadow's format (0: none)
  int32_t xexp = 0;       // the shadow's power-of-two scale e_x (fp16)
  double rmax = 0, rho = 0;   // max |x~ 2^-e_x - x|, max |x~ 2^-e_x - x| / |x| (measured at load, fp64)
  void *xl = nullptr;        // fp16 only: the refine pass's low half x_lo [n x d]
  // set (by a plain store from finalize, through mapped pinned memory -- no copy, no sync) once a
  // query of this index failed its level-0 certificate: the refine pass is launched from then on
  volatile int32_t *uncert_seen_host = nullptr;
  int32_t *uncert_seen_dev = nullptr;
  double rmax2 = 0, rho2 = 0;   // the same maxima after x~ + x_lo
  // vrs_search_host staging: device slots (queries in, ids / dists out) so
  // that the upload of one call overlaps the compute of the previous one; the
  // copies run on their own streams, ordered by events.
  std::mutex host_mu;
  cudaStream_t up_stream = nullptr, down_stream = nullptr;
  // (4 slots: a call's upload waits for the download of the call 4 back, so short
  // calls in a row do not chain compute -> download -> upload -> compute)
  static constexpr int kSlots = 4;
  void *slot_buf[kSlots] = {};
  size_t slot_cap[kSlots] = {};
  cudaEvent_t slot_free[kSlots] = {}, up_done[kSlots] = {}, comp_done[kSlots] = {};
  int slot_next = 0;
  int last_down = -1;     // slot of the last download issued (vrs_host_fence)
  int32_t device;
  int32_t num_sms;
};

// ---- kernel profiler (CUDA events on the launch stream) --------------------------
namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
struct ProfTotal {
  std::string name;
  double ms = 0;
  int64_t n = 0;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_pending;
std::vector<ProfTotal> g_prof_totals;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_resolve() {
  for (auto &r : g_prof_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto it = std::find_if(g_prof_totals.begin(), g_prof_totals.end(), [&](const ProfTotal &t) { return t.name == r.name; });
    if (it == g_prof_totals.end()) {
      g_prof_totals.push_back({r.name, 0, 0});
      it = g_prof_totals.end() - 1;
    }
    it->ms += ms;
    it->n += 1;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_pending.clear();
}
}  // namespace

namespace vrs {
ProfScope::ProfScope(const char *n, cudaStream_t st) : name(n), s(st) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  a = prof_event();
  cudaEventRecord(a, s);
}
ProfScope::~ProfScope() {
  if (!a) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEvent_t b = prof_event();
  cudaEventRecord(b, s);
  g_prof_pending.push_back({name, a, b});
}
}  // namespace vrs

static thread_local char g_err[512];
static thread_local int32_t g_last_path = 0;
static thread_local int32_t g_last_launches = 0;
static thread_local int32_t g_last_prec = 0;

static vrs_status fail(vrs_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return st;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) return fail(VRS_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

static bool is_device_ptr(const void *p) {
  if (p == nullptr) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static vrs_status check_device(int *dev_out, int *sms_out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int major = 0, minor = 0, sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (major != 10 || minor != 0)
    return fail(VRS_EUNSUPPORTED, "device %d is sm_%d%d; libvrs is built for sm_100a only", dev, major, minor);
  if (dev_out) *dev_out = dev;
  if (sms_out) *sms_out = sms;
  return VRS_OK;
}

// ---- scratch --------------------------------------------------------------------
struct Scratch {
  const vrs_allocator *alloc;
  cudaStream_t stream;
  void *ptr = nullptr;
  ~Scratch() {
    if (!ptr) return;
    if (alloc) alloc->free(ptr, stream, alloc->ctx);
    else cudaFreeAsync(ptr, stream);
  }
};

static constexpr uint64_t kPoolKeep = uint64_t(2) << 30;   // 2 GiB

static vrs_status scratch_alloc(Scratch &s, size_t bytes) {
  // size classes of 1/8 of a power of two: consecutive searches of different
  // shapes then reuse the stream-ordered pool's blocks instead of mapping new
  // memory (large gather buffers made that churn cost more than the search)
  bytes = std::max<size_t>(bytes, 256);
  {
    size_t p2 = 1;
    while (p2 < bytes) p2 <<= 1;
    const size_t step = std::max<size_t>(p2 / 8, 256);
    bytes = (bytes + step - 1) / step * step;
  }
  if (s.alloc) {
    s.ptr = s.alloc->alloc(bytes, s.stream, s.alloc->ctx);
    if (!s.ptr) return fail(VRS_ENOMEM, "allocator returned NULL for %zu bytes", bytes);
    return VRS_OK;
  }
  {  // keep up to kPoolKeep of freed scratch in the device's pool (consecutive searches reuse
     // it instead of mapping new memory); above that the pool returns memory to the driver at
     // the next synchronisation -- bounded, it never holds a large gather buffer for good
    static uint64_t tuned = 0;   // bit per device
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev < 64) {
      std::lock_guard<std::mutex> g(setup_mutex());
      cudaMemPool_t pool;
      if (!(tuned >> dev & 1) && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        tuned |= uint64_t(1) << dev;
      }
    }
  }
  cudaError_t e = cudaMallocAsync(&s.ptr, bytes, s.stream);
  if (e != cudaSuccess) {
    s.ptr = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? VRS_ENOMEM : VRS_ECUDA, "cudaMallocAsync(%zu): %s", bytes,
                cudaGetErrorString(e));
  }
  return VRS_OK;
}

struct Carve {
  char *base;
  size_t off = 0;
  explicit Carve(void *p) : base(static_cast<char *>(p)) {}
  template <typename T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T *p = reinterpret_cast<T *>(base + off);
    off += count * sizeof(T);
    return p;
  }
};
static size_t carve_size(std::initializer_list<size_t> parts) {
  size_t off = 0;
  for (size_t b : parts) off = ((off + 255) & ~size_t(255)) + b;
  return off + 256;
}

// ---- predicate ---------------------------------------------------------------------
static vrs_status make_pred(const vrs_index *ix, const vrs_predicate *pred, PredDev *out) {
  memset(out, 0, sizeof *out);
  if (!pred || pred->n_clauses == 0) return VRS_OK;
  if (pred->n_clauses < 0) return fail(VRS_EINVAL, "n_clauses < 0");
  if (pred->n_clauses > VRS_MAX_CLAUSES)
    return fail(VRS_EUNSUPPORTED, "%d clauses > VRS_MAX_CLAUSES (%d)", pred->n_clauses, VRS_MAX_CLAUSES);
  if (!pred->clauses) return fail(VRS_EINVAL, "clauses is NULL with n_clauses > 0");
  out->n = pred->n_clauses;
  for (int c = 0; c < pred->n_clauses; ++c) {
    const vrs_clause &cl = pred->clauses[c];
    if (cl.attr < 0 || cl.attr >= ix->n_attrs)
      return fail(VRS_ENOTFOUND, "clause %d names attribute %d; the index has %d", c, cl.attr, ix->n_attrs);
    const vrs_attr &at = ix->attrs[cl.attr];
    const int64_t tmin = at.type == VRS_ATTR_I32 ? INT32_MIN : 0;
    const int64_t tmax = at.type == VRS_ATTR_I32 ? INT32_MAX : 255;
    const int64_t lo = std::max(cl.lo, tmin), hi = std::min(cl.hi, tmax);
    out->c[c].col = at.data;
    out->c[c].type = at.type;
    if (lo > hi) {
      out->empty = 1;
      out->c[c].lo = 1;
      out->c[c].hi = 0;
    } else {
      out->c[c].lo = (int32_t)lo;
      out->c[c].hi = (int32_t)hi;
    }
  }
  return VRS_OK;
}

// The work the select kernels do for the tensor-core pass: the 16-bit query
// operand with its per-query exponent and residual (zero-padded to whole 128-row tiles).
static SelectFuse select_fuse(const vrs_index *ix, const float *queries, int64_t q, const GemmPlan &gp, bool h16,
                              void *qb, int32_t *qexp, float *rq) {
  SelectFuse f{};
  if (h16) {
    f.q_in = queries;
    f.q_out = qb;
    f.q = q;
    f.rows = (int64_t)gp.qtiles * 128;
    f.d = ix->d;
    f.fmt = ix->prec16 == VRS_PREC_FP16 ? 0 : 1;
    f.qexp = qexp;
    f.rq = rq;
  }
  return f;
}

static void slot_release(vrs_index *ix, int i) {
  if (!ix->slot_buf[i]) return;
  if (ix->has_alloc) ix->alloc.free(ix->slot_buf[i], nullptr, ix->alloc.ctx);
  else cudaFree(ix->slot_buf[i]);
  ix->slot_buf[i] = nullptr;
  ix->slot_cap[i] = 0;
}

// ---- ABI ----------------------------------------------------------------------------
extern "C" {

const char *vrs_last_error(void) { return g_err; }

void vrs_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

void vrs_profile_reset(void) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  prof_resolve();
  g_prof_totals.clear();
}

int32_t vrs_profile_read(int32_t i, const char **name, double *total_ms, int64_t *launches) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  prof_resolve();
  if (i >= 0 && i < (int32_t)g_prof_totals.size()) {
    if (name) *name = g_prof_totals[i].name.c_str();
    if (total_ms) *total_ms = g_prof_totals[i].ms;
    if (launches) *launches = g_prof_totals[i].n;
  }
  return (int32_t)g_prof_totals.size();
}
int32_t vrs_last_path(void) { return g_last_path; }
int32_t vrs_last_precision(void) { return g_last_prec; }
int32_t vrs_index_precision(const vrs_index *ix) { return ix ? (ix->xb ? ix->prec16 : VRS_PREC_TF32) : -1; }
int32_t vrs_last_launches(void) { return g_last_launches; }

int64_t vrs_pool_reserved_bytes(void) {
  int dev = 0;
  cudaMemPool_t pool;
  uint64_t v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess ||
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return (int64_t)v;
}
int64_t vrs_index_rows(const vrs_index *ix) { return ix ? ix->n : -1; }
int32_t vrs_index_dim(const vrs_index *ix) { return ix ? ix->d : -1; }

vrs_status vrs_load(const float *vectors, int64_t n, int32_t d, const vrs_attr *attrs, int32_t n_attrs,
                    int64_t row_offset, const vrs_allocator *alloc, void *cuda_stream, vrs_index **out) {
  return vrs_load_ex(vectors, n, d, attrs, n_attrs, row_offset, alloc, nullptr, cuda_stream, out);
}

vrs_status vrs_load_ex(const float *vectors, int64_t n, int32_t d, const vrs_attr *attrs, int32_t n_attrs,
                       int64_t row_offset, const vrs_allocator *alloc, const vrs_load_options *opts,
                       void *cuda_stream, vrs_index **out) {
  g_err[0] = 0;
  if (!out) return fail(VRS_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || n >= (int64_t(1) << 31)) return fail(VRS_EINVAL, "n = %lld outside [1, 2^31)", (long long)n);
  if (d < 1) return fail(VRS_EINVAL, "d = %d < 1", d);
  if (n_attrs < 0 || n_attrs > 64) return fail(VRS_EINVAL, "n_attrs = %d outside [0, 64]", n_attrs);
  if (n_attrs > 0 && !attrs) return fail(VRS_EINVAL, "attrs is NULL with n_attrs > 0");
  if (row_offset < 0) return fail(VRS_EINVAL, "row_offset < 0");
  if (alloc && (!alloc->alloc || !alloc->free)) return fail(VRS_EINVAL, "allocator without alloc/free");
  const int prec = opts ? opts->precision : VRS_PREC_DEFAULT;
  if (prec < VRS_PREC_DEFAULT || prec > VRS_PREC_FP16) return fail(VRS_EINVAL, "bad precision %d", prec);
  // 16-bit rows must be 16-byte aligned for TMA: d % 8 == 0 and a 16-byte aligned base
  const bool shadow_ok = d % 8 == 0 && ((uintptr_t)vectors & 15) == 0;
  if ((prec == VRS_PREC_BF16 || prec == VRS_PREC_FP16) && !shadow_ok)
    return fail(VRS_EUNSUPPORTED, "a 16-bit shadow needs d %% 8 == 0 and 16-byte aligned vectors (d = %d)", d);
  const bool want_shadow = prec == VRS_PREC_BF16 || prec == VRS_PREC_FP16 || (prec == VRS_PREC_DEFAULT && shadow_ok);
  const int prec16 = want_shadow ? (prec == VRS_PREC_BF16 ? VRS_PREC_BF16 : VRS_PREC_FP16) : 0;
  int dev = 0, sms = 0;
  vrs_status st = check_device(&dev, &sms);
  if (st != VRS_OK) return st;
  if (!is_device_ptr(vectors)) return fail(VRS_EINVAL, "vectors is not a device pointer");
  for (int a = 0; a < n_attrs; ++a) {
    if (attrs[a].type != VRS_ATTR_I32 && attrs[a].type != VRS_ATTR_U8)
      return fail(VRS_EINVAL, "attribute %d has bad type %d", a, (int)attrs[a].type);
    if (!is_device_ptr(attrs[a].data)) return fail(VRS_EINVAL, "attribute %d is not a device pointer", a);
  }
  vrs_index *ix = new vrs_index();
  ix->X = vectors;
  ix->n = n;
  ix->d = d;
  ix->n_attrs = n_attrs;
  for (int a = 0; a < n_attrs; ++a) ix->attrs[a] = attrs[a];
  ix->row_offset = row_offset;
  ix->has_alloc = alloc != nullptr;
  if (alloc) ix->alloc = *alloc;
  ix->device = dev;
  ix->num_sms = sms;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  // (the refine pass's x_lo: fp16 shadows, unless VRS_NO_REFINE)
  static const bool no_refine = getenv("VRS_NO_REFINE") != nullptr;
  const bool want_lo = want_shadow && prec16 == VRS_PREC_FP16 && !no_refine;
  const size_t bytes = carve_size({(size_t)n * 4, (size_t)n * 4, 16, 32, want_shadow ? (size_t)n * d * 2 : 0,
                                   want_lo ? (size_t)n * d * 2 : 0});
  void *mem = nullptr;
  if (alloc) {
    mem = alloc->alloc(bytes, cuda_stream, alloc->ctx);
    if (!mem) {
      delete ix;
      return fail(VRS_ENOMEM, "allocator returned NULL for %zu bytes", bytes);
    }
  } else if (cudaMalloc(&mem, bytes) != cudaSuccess) {
    cudaGetLastError();
    delete ix;
    return fail(VRS_ENOMEM, "cudaMalloc(%zu) failed", bytes);
  }
  Carve cv(mem);
  ix->nx2 = cv.take<float>(n);
  ix->inv_nx = cv.take<float>(n);
  int32_t *zf = cv.take<int32_t>(4);   // [0] zero-norm row flag, [1] max |x|^2, [2] max |x_t| (float bits)
  unsigned long long *res = cv.take<unsigned long long>(4);   // shadow residual maxima (double bits)
  ix->xb = want_shadow ? cv.take<char>((size_t)n * d * 2) : nullptr;
  ix->xl = want_lo ? cv.take<char>((size_t)n * d * 2) : nullptr;
  ix->prec16 = prec16;
  int32_t flags[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemsetAsync(zf, 0, 16, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(res, 0, 32, stream);
  if (e == cudaSuccess) e = launch_norms(vectors, n, d, ix->nx2, ix->inv_nx, zf, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(flags, zf, 16, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess && ix->xb) {
    // fp16: one power of two for the whole corpus puts max |x_t| into [2^14, 2^15)
    // (convert16.cuh scale_exp16); bf16 needs no scaling
    float amax;
    memcpy(&amax, &flags[2], 4);
    if (prec16 == VRS_PREC_FP16 && amax > 0.f && std::isfinite(amax))
      ix->xexp = std::max(-120, std::min(120, 14 - ilogbf(amax)));
    unsigned long long r2[4] = {0, 0, 0, 0};
    e = launch_shadow(vectors, n, d, ix->xexp, prec16 == VRS_PREC_FP16 ? 0 : 1, ix->xb, ix->xl, ix->nx2, res, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(r2, res, 32, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    memcpy(&ix->rmax, &r2[0], 8);
    memcpy(&ix->rho, &r2[1], 8);
    memcpy(&ix->rmax2, &r2[2], 8);
    memcpy(&ix->rho2, &r2[3], 8);
  }
  if (e != cudaSuccess) {
    vrs_free(ix);
    return fail(VRS_ECUDA, "vrs_load norms / shadow: %s", cudaGetErrorString(e));
  }
  ix->has_zero_row = flags[0];
  if (ix->xl) {
    int32_t *h = nullptr;
    if (cudaHostAlloc(&h, 4, cudaHostAllocMapped) == cudaSuccess) {
      *h = 0;
      void *dptr = nullptr;
      if (cudaHostGetDevicePointer(&dptr, h, 0) == cudaSuccess) {
        ix->uncert_seen_host = h;
        ix->uncert_seen_dev = static_cast<int32_t *>(dptr);
      } else {
        cudaFreeHost(h);
      }
    }
    cudaGetLastError();
  }
  {
    float m2;
    memcpy(&m2, &flags[1], 4);
    ix->xmax = sqrtf(m2) * (1.0f + 1e-6f);
  }
  *out = ix;
  return VRS_OK;
}

vrs_status vrs_free(vrs_index *ix) {
  if (!ix) return VRS_OK;
  if (ix->up_stream) {
    cudaStreamSynchronize(ix->up_stream);
    cudaStreamSynchronize(ix->down_stream);
    for (int i = 0; i < vrs_index::kSlots; ++i) {
      slot_release(ix, i);
      cudaEventDestroy(ix->slot_free[i]);
      cudaEventDestroy(ix->up_done[i]);
      cudaEventDestroy(ix->comp_done[i]);
    }
    cudaStreamDestroy(ix->up_stream);
    cudaStreamDestroy(ix->down_stream);
  }
  if (ix->nx2) {
    if (ix->has_alloc) ix->alloc.free(ix->nx2, nullptr, ix->alloc.ctx);
    else cudaFree(ix->nx2);
  }
  if (ix->uncert_seen_host) cudaFreeHost(const_cast<int32_t *>(ix->uncert_seen_host));
  delete ix;
  return VRS_OK;
}

// The X_sel copy buffer above 1 GiB is also capped at half the device's free memory
// (selections that do not fit then stream masked -- the same result).
// (cudaMemGetInfo costs ~100 us: its answer is reused for 50 ms per device)
static int64_t cap_by_free_memory(int64_t rows, int64_t row_bytes) {
  if (rows * row_bytes <= (int64_t(1) << 30)) return rows;
  static std::mutex mu;
  static int64_t cached_free[64];
  static std::chrono::steady_clock::time_point when[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) {
    cudaGetLastError();
    return rows;
  }
  int64_t fr;
  {
    std::lock_guard<std::mutex> g(mu);
    const auto now = std::chrono::steady_clock::now();
    if (cached_free[dev] <= 0 || now - when[dev] > std::chrono::milliseconds(50)) {
      size_t f = 0, tot = 0;
      if (cudaMemGetInfo(&f, &tot) != cudaSuccess) {
        cudaGetLastError();
        return rows;
      }
      cached_free[dev] = (int64_t)f;
      when[dev] = now;
    }
    fr = cached_free[dev];
  }
  return std::max<int64_t>(1, std::min<int64_t>(rows, (fr / 2) / row_bytes));
}

// ---- row delivery plan of the tensor-core pass ("Row delivery") ------
// A selection is delivered gathered (only its rows; late materialization) iff
// N_sel <= gather_cap -- decided on the device from the selection count -- else every
// row streams by TMA with the unqualified ones masked.  Gathered rows reach the pass
// either through an X_sel copy (gather_copy_kernel, then TMA tiles; 2 x the row bytes,
// but read once per query tile) or fetched by id with coalesced cp.async straight into
// the swizzled stages (no copy; each query tile re-reads them) -- the latter for at most
// cp_qtiles query tiles and selections of >= cp_min_bytes.  Break-even selectivities
// (B200 measurements, profiles/r02_rowplan_*.txt): masked rows stream at ~6.9 TB/s,
// cp.async-gathered ones at ~5 TB/s per query tile, copied ones cost a read + write.
struct RowPlan {
  int64_t gather_cap;      // gathered iff N_sel <= gather_cap (0: always masked)
  int64_t xsel_rows;       // rows of the X_sel copy buffer
  int64_t cp_min_bytes;    // cp.async iff gathered and N_sel * row_bytes >= this (INT64_MAX: never) ...
  int64_t cp_min_rows;     // ... or N_sel >= this (cp_fetch)
};
static RowPlan row_plan(int64_t q, int32_t qtiles, int64_t n, int64_t row_bytes, int rows_req, bool identity) {
  static const int cp_qtiles = getenv("VRS_CP_QTILES") ? atoi(getenv("VRS_CP_QTILES")) : 2;
  static const int64_t cp_min = (getenv("VRS_CP_MIN_MB") ? (int64_t)atoll(getenv("VRS_CP_MIN_MB")) : 64) << 20;
  static const double cp_frac = getenv("VRS_GATHER_CP_FRAC") ? atof(getenv("VRS_GATHER_CP_FRAC")) : 0.7;
  static const bool direct = getenv("VRS_GATHER4") != nullptr || getenv("VRS_CPGATHER") != nullptr;
  // (cp.async also for >= 2 x 148 row tiles of any size: enough tiles that the by-id fetch,
  // ~38 GB/s per SM with two producer warps, runs on every SM -- C2 s = 10 %, Q <= 256: 25.6 MB,
  // 4-6 us faster than the copy; fewer tiles leave most SMs idle: C4 s = 0.1 %, Q = 1, 25 tiles:
  // the copy is 10 us faster; r02_planner_c2.txt, r02_planner_c4.txt)
  static const int64_t cp_min_rows = getenv("VRS_CP_MIN_ROWS") ? atoll(getenv("VRS_CP_MIN_ROWS"))
                                                               : int64_t(2) * kSmCountB200 * 256;
  RowPlan r{0, 0, INT64_MAX, INT64_MAX};
  if (identity || rows_req == VRS_ROWS_MASKED) return r;
  const bool cp = qtiles <= cp_qtiles && getenv("VRS_NO_CPGATHER") == nullptr;
  int64_t cap = q >= 1024 ? n * 9 / 10 : q >= 256 ? n * 9 / 20 : n / 3;
  // (masked and cp.async-gathered rows are both re-read per query tile: the break-even
  // selectivity is the rate ratio, ~0.7, whatever the tile count)
  if (cp) cap = std::max<int64_t>(cap, (int64_t)(n * cp_frac));
  if (rows_req == VRS_ROWS_GATHER) cap = n;
  r.gather_cap = cap;
  if (direct) return r;   // (VRS_GATHER4 / VRS_CPGATHER: rows by id from X, no buffer; tc_prepare)
  r.cp_min_bytes = cp ? cp_min : INT64_MAX;
  r.cp_min_rows = cp ? cp_min_rows : INT64_MAX;
  int64_t buf = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(16) << 30) / row_bytes));
  if (cp)   // copies stay below cp_min and cp_min_rows
    buf = std::min<int64_t>(buf, std::max<int64_t>(1, std::min((cp_min - 1) / row_bytes, cp_min_rows - 1)));
  r.xsel_rows = cap_by_free_memory(buf, row_bytes);
  if (!cp) r.gather_cap = std::min(r.gather_cap, r.xsel_rows);
  return r;
}

static int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// The selection over-fetches k' candidates for the exact re-score: k + 16 for k <= 16,
// else the power of two >= k + 16 -- the lists keep that many per (list, query) anyway,
// and the wider margin lets the certificate hold without the fallback (
// C4 k = 100: 116 certified 99 %, 128 100 %; C5 k = 50 -> 128).
// wide: the index has seen a level-0 certificate fail (its mapped flag) -- data whose
// k-th and k'-th keys crowd within the fp16 bound (C5: clustered, cosine); twice the
// over-fetch (<= 256) certifies most queries at level 0 instead of sending them through the
// refine pass (C5: 89 -> 98 % certified at level 0, 3.44 -> 3.18 ms per step,
// r02_kprime_c5_ab.txt); VRS_KPRIME_WIDE=0 disables
static int kprime_of(int k, bool wide = false) {
  static const bool old = getenv("VRS_KPRIME_K16") != nullptr;   // (A/B only: r01's k + 16)
  static const int forced = getenv("VRS_KPRIME") ? atoi(getenv("VRS_KPRIME")) : 0;   // (A/B only)
  static const bool wide_ok = !getenv("VRS_KPRIME_WIDE") || atoi(getenv("VRS_KPRIME_WIDE")) > 0;
  if (forced > 0) return std::max(k + 1, std::min(256, forced));
  const int base = (old || k <= 16) ? k + 16   // (small k: the margin of 16 already exceeds k; C2 k' = 26: +3 % vs 32)
                                    : std::max(32, pow2_at_least(k + 16));
  return wide && wide_ok ? std::max(base, std::min(256, 2 * base)) : base;
}

static vrs_status check_precision(const vrs_index *ix, int prec_req) {
  if (prec_req < VRS_PREC_DEFAULT || prec_req > VRS_PREC_FP16) return fail(VRS_EINVAL, "bad precision option");
  if ((prec_req == VRS_PREC_BF16 || prec_req == VRS_PREC_FP16) && ix->prec16 != prec_req)
    return fail(VRS_EUNSUPPORTED, "the index has no %s shadow", prec_req == VRS_PREC_BF16 ? "bf16" : "fp16");
  return VRS_OK;
}

// Error-bound constants of the selection pass (vrs_internal.cuh key_error_bound).
static KeyBound key_bound(const vrs_index *ix, bool gemm, bool h16) {
  KeyBound b{};
  b.kind = !gemm ? (h16 ? KEY_H16_FFMA : KEY_FP32) : (h16 ? KEY_H16 : KEY_TF32);
  b.d = ix->d;
  b.rmax = ix->rmax;
  b.rho = ix->rho;
  b.xmax = ix->xmax;
  b.rmax2 = ix->rmax2;
  b.rho2 = ix->rho2;
  return b;
}

vrs_status vrs_search_ex(vrs_index *ix, const float *queries, int64_t q, int32_t d, const vrs_predicate *pred,
                         int32_t k, vrs_metric metric, int64_t *ids, float *dists,
                         const vrs_search_options *opts, void *cuda_stream) {
  g_err[0] = 0;
  g_last_launches = 0;
  if (!ix) return fail(VRS_EINVAL, "index is NULL");
  if (q < 0) return fail(VRS_EINVAL, "q < 0");
  if (d != ix->d) return fail(VRS_EINVAL, "d = %d differs from the loaded d = %d", d, ix->d);
  if (k < 1) return fail(VRS_EINVAL, "k = %d < 1", k);
  if (metric != VRS_L2 && metric != VRS_IP && metric != VRS_COSINE)
    return fail(VRS_EINVAL, "bad metric %d", (int)metric);
  const int path_req = opts ? opts->path : VRS_PATH_AUTO;
  const int rows_req = opts ? opts->rows : VRS_ROWS_AUTO;
  if (path_req < VRS_PATH_AUTO || path_req > VRS_PATH_GEMM) return fail(VRS_EINVAL, "bad path option");
  if (rows_req < VRS_ROWS_AUTO || rows_req > VRS_ROWS_MASKED) return fail(VRS_EINVAL, "bad rows option");
  const int prec_req = opts ? opts->precision : VRS_PREC_DEFAULT;
  vrs_status st = check_precision(ix, prec_req);
  if (st != VRS_OK) return st;
  const bool use16 = ix->xb && prec_req != VRS_PREC_TF32;   // (16-bit shadow: fp16 or bf16)
  PredDev pd;
  st = make_pred(ix, pred, &pd);
  if (st != VRS_OK) return st;
  if (k > VRS_K_MAX) return fail(VRS_EUNSUPPORTED, "k = %d > VRS_K_MAX (%d)", k, VRS_K_MAX);
  if (metric == VRS_COSINE && ix->has_zero_row)
    return fail(VRS_EDEGENERATE, "COSINE over a corpus with a zero-norm row");
  if (q == 0) return VRS_OK;
  if (!is_device_ptr(queries) || !is_device_ptr(ids) || !is_device_ptr(dists))
    return fail(VRS_EINVAL, "queries / ids / dists must be device pointers");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != ix->device) return fail(VRS_EINVAL, "current device %d differs from the index device %d", dev, ix->device);

  cudaStream_t stream = (cudaStream_t)cuda_stream;
  // over-fetch for the exact re-score; wider once the index has seen a
  // level-0 certificate fail on the 16-bit path
  const bool seen_uncert = ix->xb && prec_req != VRS_PREC_TF32 && ix->uncert_seen_host && *ix->uncert_seen_host != 0;
  const int32_t kprime = kprime_of(k, seen_uncert);
  const int kpe = std::max(64, pow2_at_least(kprime));
  const bool identity = (pd.n == 0);
  const int64_t n = ix->n;

  // path choice (A16: per-tuple for small batches, tensor formulation for large ones)
  int path = path_req;
  GemmPlan gp{0, 0, 0, 1};
  // the TMA paths need 16-byte aligned rows and bases
  const bool tma_ok = (((uintptr_t)queries | (uintptr_t)ix->X) & 15) == 0;
  if (path != VRS_PATH_SCAN && tma_ok) gp = gemm_plan(q, d, n, kprime, ix->num_sms, use16);
  // (measured on C2: the tensor-core pass over the 16-bit shadow is HBM-bound and beats
  // the fp32 FFMA scan already at q = 1 -- it reads half the bytes)
  if (path == VRS_PATH_AUTO) path = gp.ok ? VRS_PATH_GEMM : VRS_PATH_SCAN;
  if (path == VRS_PATH_GEMM && !gp.ok) return fail(VRS_EUNSUPPORTED, "tensor-core path does not support this shape");


  int qg = 0, P = 0;
  if (path == VRS_PATH_SCAN) {
    qg = scan_query_group(q, d, kpe);
    if (qg == 0) return fail(VRS_EUNSUPPORTED, "d = %d too large for the scan path", d);
    const int64_t gy = (q + qg - 1) / qg;
    const int64_t want = std::max<int64_t>(1, ix->num_sms / gy);
    P = (int)std::min<int64_t>(want, std::max<int64_t>(1, (n + 255) / 256));
  } else {
    P = gp.P;
  }
  const size_t nwords = (size_t)((n + 31) / 32);
  const size_t part_entries = path == VRS_PATH_SCAN ? (size_t)P * q * kprime : 0;
  Scratch scr{ix->has_alloc ? &ix->alloc : nullptr, stream};
  // Selectivity-driven row delivery of the tensor-core pass (decided on the
  // device from the selection count): the selection is materialised densely
  // ("gathered", late materialization) iff N_sel <= xsel_cap, else full row
  // tiles stream with unqualified rows masked.  Gathering costs a copy of the
  // selected rows (2 x row bytes each); masking costs MMA / TMEM work and HBM
  // reads on the unselected rows.  Break-even (C2/C3/C4 measurements, DESIGN.md
  // Sec. 6): selectivity 1/3 while the pass is HBM-bound (q < 256), ~0.45 at
  // q = 256, 0.9 once it is tensor / TMEM-bound (q >= 1024).  The buffer holds
  // at most 16 GiB of rows.
  const int64_t row_bytes = (int64_t)d * (use16 ? 2 : 4);
  const size_t qpad_bytes = (size_t)gp.qtiles * 128 * d * 2;   // 16-bit queries, whole 128-row tiles
  const RowPlan rp = path == VRS_PATH_GEMM ? row_plan(q, gp.qtiles, n, row_bytes, rows_req, identity)
                                           : RowPlan{0, 0, INT64_MAX, INT64_MAX};
  const int64_t xsel_cap = rp.gather_cap;
  const int64_t xsel_rows = rp.xsel_rows;   // rows of the X_sel buffer
  // VRS_SELECT_LOCAL=1: one-kernel selection (chunk-local ids) + select_finish (count, dense
  // ids, gathered rows in one launch) instead of select_count + select_scatter + gather_copy.
  // Measured: equal on C2's small cells, 10-20 % slower gathers on C5 -- so opt-in.
  static const bool want_local = getenv("VRS_SELECT_LOCAL") != nullptr;
  const bool sel_local = want_local && path == VRS_PATH_GEMM && !identity && select_chunks(n) <= kSelFinishMaxChunks;
  const size_t local_ids = sel_local ? (size_t)select_chunks(n) * kSelChunkRows : 0;
  // certificate + exact fallback: per query the exponent / residual of
  // the 16-bit operand, the certificate, finalize's k-th sort key, a group counter; the
  // fallback's per-(item, query) slots of k results
  const int ex_qg = exact_group_size(d, k);
  // the refine pass for batches of >= 128 queries on the fp16 tensor-core
  // path (below that the exact fallback's row passes cost less than a tensor pass's launch chain)
  // -- and only once the index has seen a level-0 certificate fail (the flag finalize sets): an
  // index whose data always certifies pays no launches for it (C2: 8 cells x 3 launches);
  // VRS_REFINE=always / never for A/B.  Correctness never depends on it: the exact fallback
  // recomputes whatever stays uncertified.
  static const int refine_qmin = getenv("VRS_REFINE_QMIN") ? atoi(getenv("VRS_REFINE_QMIN")) : 128;
  static const int refine_mode = !getenv("VRS_REFINE") ? 0 : (strcmp(getenv("VRS_REFINE"), "always") == 0 ? 1 : -1);
  const bool refine_seen = refine_mode == 1 || (refine_mode == 0 && ix->uncert_seen_host && *ix->uncert_seen_host != 0);
  const bool refine = path == VRS_PATH_GEMM && use16 && ix->xl != nullptr && q >= refine_qmin && refine_seen &&
                      (prec_req == VRS_PREC_DEFAULT || prec_req == VRS_PREC_FP16);
  const int32_t rf_dpad = (d + 63) / 64 * 64;
  // the refine's X_sel_lo (x_lo rows of the selection, beside level 0's X_sel of x_hi rows),
  // when both fit the free-memory share the X_sel alone is capped by; else cp.async by id
  const int64_t xlo_rows = refine && xsel_rows > 0 && cap_by_free_memory(xsel_rows, 2 * row_bytes) == xsel_rows
                               ? xsel_rows : 0;
  const size_t rf_rows = (size_t)gp.qtiles * 128;
  const int64_t ex_items = exact_items_max(q, ex_qg);
  const size_t ex_slots = (size_t)ex_items * ex_qg;
  const size_t bytes = carve_size({nwords * 4, identity ? 0 : (size_t)n * 4, 8, select_scratch_bytes(n),
                                   local_ids * 4, part_entries * 4, part_entries * 4,
                                   path == VRS_PATH_GEMM ? gemm_scratch_bytes(gp, q, kprime) : 0,
                                   (size_t)(xsel_rows * row_bytes), (size_t)xsel_rows * 4,
                                   use16 && path == VRS_PATH_GEMM ? qpad_bytes : 0,
                                   (size_t)q * 4, (size_t)q * 4, (size_t)q, (size_t)q * 8, (size_t)q * 4,
                                   ex_slots * k * 8, ex_slots * k * 8, ex_slots * 4,
                                   refine ? (size_t)q * 4 : 0, refine ? (size_t)16 : 0, refine ? rf_rows * 2 * (size_t)rf_dpad * 2 : 0,
                                   refine ? (size_t)q * 4 : 0, refine ? (size_t)q * 4 : 0, refine ? (size_t)q * 4 : 0,
                                   refine ? (size_t)q * 4 : 0, (size_t)(xlo_rows * row_bytes)});
  st = scratch_alloc(scr, bytes);
  if (st != VRS_OK) return st;
  Carve cv(scr.ptr);
  uint32_t *bitmap = cv.take<uint32_t>(nwords);
  int32_t *sel_ids = identity ? nullptr : cv.take<int32_t>((size_t)n);
  int64_t *count = cv.take<int64_t>(1);
  void *sel_scratch = cv.take<char>(select_scratch_bytes(n));
  int32_t *ids_local = sel_local ? cv.take<int32_t>(local_ids) : nullptr;
  float *part_key = cv.take<float>(part_entries);
  int32_t *part_id = cv.take<int32_t>(part_entries);
  void *gemm_scr = path == VRS_PATH_GEMM ? cv.take<char>(gemm_scratch_bytes(gp, q, kprime)) : nullptr;
  void *xsel = xsel_rows > 0 ? cv.take<char>((size_t)(xsel_rows * row_bytes)) : nullptr;
  float *xsel_norm = xsel_rows > 0 ? cv.take<float>((size_t)xsel_rows) : nullptr;
  void *qb = use16 && path == VRS_PATH_GEMM ? cv.take<char>(qpad_bytes) : nullptr;
  int32_t *qexp = cv.take<int32_t>((size_t)q);
  float *rq = cv.take<float>((size_t)q);
  uint8_t *cert = cv.take<uint8_t>((size_t)q);
  double *skey = cv.take<double>((size_t)q);
  int32_t *gcnt = cv.take<int32_t>((size_t)q);
  double *slot_key = cv.take<double>(ex_slots * k);
  int64_t *slot_id = cv.take<int64_t>(ex_slots * k);
  int32_t *slot_cnt = cv.take<int32_t>(ex_slots);
  int32_t *rf_qlist = refine ? cv.take<int32_t>((size_t)q) : nullptr;
  int32_t *rf_count = refine ? cv.take<int32_t>(4) : nullptr;
  uint16_t *rf_qr = refine ? cv.take<uint16_t>(rf_rows * 2 * rf_dpad) : nullptr;
  int32_t *rf_qexp = refine ? cv.take<int32_t>((size_t)q) : nullptr;
  float *rf_rqa = refine ? cv.take<float>((size_t)q) : nullptr;
  float *rf_rq2 = refine ? cv.take<float>((size_t)q) : nullptr;
  uint32_t *rf_gtau = refine ? cv.take<uint32_t>((size_t)q) : nullptr;
  void *rf_xsel_lo = xlo_rows > 0 ? cv.take<char>((size_t)(xlo_rows * row_bytes)) : nullptr;
  const bool h16 = use16 && path == VRS_PATH_GEMM;   // (16-bit query operand of the tensor-core pass)

  int launches = 0;
  GemmArgs gemm_args{};   // (the tensor-core pass's arguments, reused by the refine pass)
  void *gemm_scr_keep = gemm_scr;
  FinalizeArgs f{part_key, part_id, nullptr, P, kprime, kprime, 1, nullptr, SplitInfo{}, kprime, q, ix->X, d,
                 queries, (int32_t)metric, k, ix->row_offset, ids, dists};
  if (path == VRS_PATH_SCAN) {
    if (!identity) {
      ProfScope ps("select", stream);
      CUDA_TRY(launch_select(pd, n, bitmap, sel_ids, count, sel_scratch, stream, &launches));
    }
    ScanArgs a{ix->X, n, d, sel_ids, count, queries, q, ix->nx2, ix->inv_nx, (int32_t)metric, kprime,
               part_key, part_id, P};
    if (use16) {   // the scan streams the 16-bit shadow (half the bytes) unless TF32 (= fp32 rows) is asked for
      a.Xh = ix->xb;
      a.fmt16 = ix->prec16 == VRS_PREC_FP16 ? 0 : 1;
      a.xexp = ix->xexp;
    }
    ProfScope ps("scan", stream);
    CUDA_TRY(launch_scan(a, qg, kpe, stream, &launches));
  } else {
    // tensor-core path: gathered selection or bitmap-masked full tiles, chosen on the device
    const int32_t rows_mode = rows_req == VRS_ROWS_MASKED ? 1 : (rows_req == VRS_ROWS_GATHER ? 2 : 0);
    if (!identity) {   // (the 16-bit query conversion rides along)
      ProfScope ps("select", stream);
      const SelectFuse fz = select_fuse(ix, queries, q, gp, use16, qb, qexp, rq);
      if (sel_local) CUDA_TRY(launch_select_local(pd, n, bitmap, ids_local, sel_scratch, stream, &launches, &fz));
      else CUDA_TRY(launch_select(pd, n, bitmap, sel_ids, count, sel_scratch, stream, &launches, &fz));
    }
    GemmArgs a{ix->X, n, d, sel_ids, count, identity ? nullptr : bitmap, rows_mode, xsel, xsel_cap, xsel_norm,
               queries, q, ix->nx2, ix->inv_nx, (int32_t)metric, kprime, part_key, part_id, P,
               use16 ? 1 : 0, ix->xb, qb, identity ? 0 : 1};
    a.fmt16 = ix->prec16 == VRS_PREC_FP16 ? 0 : 1;
    a.xexp = ix->xexp;
    a.qexp = qexp;
    a.rq = rq;
    a.cp_min_bytes = rp.cp_min_bytes;
    a.cp_min_rows = rp.cp_min_rows;
    a.ids_local = ids_local;
    gemm_args = a;
    a.chunk_count = sel_local ? static_cast<const uint32_t *>(sel_scratch) : nullptr;
    {
      ProfScope ps("gemm", stream);
      CUDA_TRY(launch_gemm(a, gp, gemm_scr, stream, &launches));
    }
    const GemmLists gl = gemm_lists(a, gp, gemm_scr);
    f.key = gl.key;
    f.id = gl.id;
    f.cnt = gl.cnt;
    f.lists = gl.lists;
    f.stride = gl.stride;
    f.kread = 0;
    f.sorted = 0;
    f.gtau = gl.gtau;
    f.split = gl.split;
  }
  // the certificate (finalize) and its fallback (exact.cu): every query's result is the
  // exact top-k of the definition -- no host synchronisation
  f.kb = key_bound(ix, path == VRS_PATH_GEMM, use16);
  f.qexp = h16 ? qexp : nullptr;
  f.rq = h16 ? rq : nullptr;
  f.xexp = h16 ? ix->xexp : 0;
  f.cert = cert;
  f.sk = skey;
  f.gcnt = gcnt;
  f.stats = opts ? reinterpret_cast<unsigned long long *>(opts->stats) : nullptr;
  f.uncert_seen = h16 ? ix->uncert_seen_dev : nullptr;
  {
    ProfScope ps("finalize", stream);
    CUDA_TRY(launch_finalize(f, stream, &launches));
  }
  if (refine) {   // level 1: the uncertified queries re-selected with split-fp16 keys, finalized again
    RefineArgs ra{cert, skey, queries, q, d, rf_dpad, (int32_t)metric, key_bound(ix, true, true), ix->xexp,
                  (int64_t)rf_rows, rf_qlist, rf_count, rf_qr, rf_qexp, rf_rqa, rf_rq2, rf_gtau};
    ra.kb.kind = KEY_H16X3;
    ra.gather_cap = rows_req == VRS_ROWS_MASKED ? 0 : (rows_req == VRS_ROWS_GATHER ? n : n * 7 / 10);
    ra.xsel_lo = rf_xsel_lo;
    {
      ProfScope ps("refine", stream);
      CUDA_TRY(launch_refine(ra, gemm_args, gp, gemm_scr_keep, ix->xl, stream, &launches));
    }
    FinalizeArgs f2 = f;
    f2.gtau = rf_gtau;
    f2.kb = ra.kb;
    f2.qexp = rf_qexp;
    f2.rq = rf_rqa;
    f2.rq2 = rf_rq2;
    f2.qmap = rf_qlist;
    f2.qcount = rf_count;
    f2.fold_qtiles = gp.qtiles;
    ProfScope ps("refine.finalize", stream);
    CUDA_TRY(launch_finalize(f2, stream, &launches));
  }
  static const bool no_fallback = getenv("VRS_NO_FALLBACK") != nullptr;   // (A/B timing only: results unverified)
  if (!no_fallback) {
    ExactArgs ea{cert, skey, gcnt, ix->X, d, n, identity ? nullptr : sel_ids, count, queries, q, (int32_t)metric, k,
                 ix->row_offset, (double)ix->xmax, ix->nx2, ix->inv_nx, ids, dists, slot_key, slot_id, slot_cnt, ex_qg};
    ea.stats = f.stats;
    ProfScope ps("exact", stream);
    CUDA_TRY(launch_exact(ea, stream, &launches));
  }
  g_last_path = path;
  g_last_prec = use16 ? ix->prec16 : (path == VRS_PATH_GEMM ? VRS_PREC_TF32 : VRS_PREC_DEFAULT);
  g_last_launches = launches;
  return VRS_OK;
}

vrs_status vrs_search(vrs_index *ix, const float *queries, int64_t q, int32_t d, const vrs_predicate *pred,
                      int32_t k, vrs_metric metric, int64_t *ids, float *dists, void *cuda_stream) {
  return vrs_search_ex(ix, queries, q, d, pred, k, metric, ids, dists, nullptr, cuda_stream);
}

vrs_status vrs_range_search(vrs_index *ix, const float *queries, int64_t q, int32_t d, const vrs_predicate *pred,
                            double tau, vrs_metric metric, int64_t capacity, int64_t *offsets, int64_t *ids,
                            float *dists, int64_t *total, const vrs_search_options *opts, void *cuda_stream) {
  g_err[0] = 0;
  g_last_launches = 0;
  if (!ix) return fail(VRS_EINVAL, "index is NULL");
  if (!total) return fail(VRS_EINVAL, "total is NULL");
  if (q < 0) return fail(VRS_EINVAL, "q < 0");
  if (d != ix->d) return fail(VRS_EINVAL, "d = %d differs from the loaded d = %d", d, ix->d);
  if (metric != VRS_L2 && metric != VRS_IP && metric != VRS_COSINE)
    return fail(VRS_EINVAL, "bad metric %d", (int)metric);
  if (tau != tau) return fail(VRS_EINVAL, "tau is NaN");
  if (capacity < 0) return fail(VRS_EINVAL, "capacity < 0");
  const int rows_req = opts ? opts->rows : VRS_ROWS_AUTO;
  if (rows_req < VRS_ROWS_AUTO || rows_req > VRS_ROWS_MASKED) return fail(VRS_EINVAL, "bad rows option");
  const int prec_req = opts ? opts->precision : VRS_PREC_DEFAULT;
  vrs_status st = check_precision(ix, prec_req);
  if (st != VRS_OK) return st;
  const bool use16 = ix->xb && prec_req != VRS_PREC_TF32;   // (16-bit shadow: fp16 or bf16)
  PredDev pd;
  st = make_pred(ix, pred, &pd);
  if (st != VRS_OK) return st;
  if (metric == VRS_COSINE && ix->has_zero_row)
    return fail(VRS_EDEGENERATE, "COSINE over a corpus with a zero-norm row");
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  if (!is_device_ptr(offsets)) return fail(VRS_EINVAL, "offsets must be a device pointer");
  if (q == 0) {
    *total = 0;
    CUDA_TRY(cudaMemsetAsync(offsets, 0, 8, stream));
    return VRS_OK;
  }
  if (!is_device_ptr(queries)) return fail(VRS_EINVAL, "queries must be a device pointer");
  if (capacity > 0 && (!is_device_ptr(ids) || !is_device_ptr(dists)))
    return fail(VRS_EINVAL, "ids / dists must be device pointers");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != ix->device) return fail(VRS_EINVAL, "current device %d differs from the index device %d", dev, ix->device);
  const bool tma_ok = (((uintptr_t)queries | (uintptr_t)ix->X) & 15) == 0;
  const int64_t n = ix->n;
  GemmPlan gp{0, 0, 0, 1};
  if (tma_ok) gp = gemm_plan(q, d, n, 32, ix->num_sms, false);   // (range passes: no CTA pairs)
  if (!gp.ok)
    return fail(VRS_EUNSUPPORTED, "range search runs on the tensor-core path: d %% 4 == 0 and 16-byte aligned rows");
  const bool identity = (pd.n == 0);
  const size_t nwords = (size_t)((n + 31) / 32);
  const int64_t row_bytes = (int64_t)d * (use16 ? 2 : 4);
  const size_t qpad_bytes = (size_t)gp.qtiles * 128 * d * 2;
  const RowPlan rp = row_plan(q, gp.qtiles, n, row_bytes, rows_req, identity);   // (as in vrs_search_ex)
  const int64_t xsel_cap = rp.gather_cap;
  const int64_t xsel_rows = rp.xsel_rows;
  const int L = kListsPerSplit * gp.P;
  Scratch scr{ix->has_alloc ? &ix->alloc : nullptr, stream};
  static const bool want_local = getenv("VRS_SELECT_LOCAL") != nullptr;   // (as in vrs_search_ex)
  const bool sel_local = want_local && !identity && select_chunks(n) <= kSelFinishMaxChunks;
  const size_t local_ids = sel_local ? (size_t)select_chunks(n) * kSelChunkRows : 0;
  st = scratch_alloc(scr, carve_size({nwords * 4, identity ? 0 : (size_t)n * 4, 8, select_scratch_bytes(n), local_ids * 4,
                                      (size_t)(xsel_rows * row_bytes), (size_t)xsel_rows * 4, use16 ? qpad_bytes : 0,
                                      (size_t)q * 4,
                                      (size_t)L * q * 4, ((size_t)L * q + 1) * 8, (size_t)q * 4, (size_t)q * 4,
                                      (size_t)q * 4}));
  if (st != VRS_OK) return st;
  Carve cv(scr.ptr);
  uint32_t *bitmap = cv.take<uint32_t>(nwords);
  int32_t *sel_ids = identity ? nullptr : cv.take<int32_t>((size_t)n);
  int64_t *count = cv.take<int64_t>(1);
  void *sel_scratch = cv.take<char>(select_scratch_bytes(n));
  int32_t *ids_local = sel_local ? cv.take<int32_t>(local_ids) : nullptr;
  void *xsel = xsel_rows > 0 ? cv.take<char>((size_t)(xsel_rows * row_bytes)) : nullptr;
  float *xsel_norm = xsel_rows > 0 ? cv.take<float>((size_t)xsel_rows) : nullptr;
  void *qb = use16 ? cv.take<char>(qpad_bytes) : nullptr;
  int32_t *qexp = cv.take<int32_t>((size_t)q);
  float *rq = cv.take<float>((size_t)q);
  RangeState r;
  r.gtau = cv.take<uint32_t>((size_t)q);
  r.cand_cnt = cv.take<int32_t>((size_t)L * q);
  r.coff = cv.take<int64_t>((size_t)L * q + 1);
  r.kept = cv.take<int32_t>((size_t)q);
  r.tau = tau;
  r.kb = key_bound(ix, true, use16);
  r.offsets = offsets;
  r.ids = ids;
  r.dists = dists;
  r.row_offset = ix->row_offset;
  struct TcGuard {
    TcLaunch *t;
    ~TcGuard() { range_tc_free(t); }
  } guard{range_tc_alloc()};
  r.tc = guard.t;
  int launches = 0;
  const int32_t rows_mode = rows_req == VRS_ROWS_MASKED ? 1 : (rows_req == VRS_ROWS_GATHER ? 2 : 0);
  if (!identity) {
    const SelectFuse fz = select_fuse(ix, queries, q, gp, use16, qb, qexp, rq);
    if (sel_local) CUDA_TRY(launch_select_local(pd, n, bitmap, ids_local, sel_scratch, stream, &launches, &fz));
    else CUDA_TRY(launch_select(pd, n, bitmap, sel_ids, count, sel_scratch, stream, &launches, &fz));
  }
  GemmArgs a{ix->X, n, d, sel_ids, count, identity ? nullptr : bitmap, rows_mode, xsel, xsel_cap, xsel_norm,
             queries, q, ix->nx2, ix->inv_nx, (int32_t)metric, 32, nullptr, nullptr, gp.P,
             use16 ? 1 : 0, ix->xb, qb, identity ? 0 : 1};
  a.fmt16 = ix->prec16 == VRS_PREC_FP16 ? 0 : 1;
  a.xexp = ix->xexp;
  a.qexp = qexp;
  a.rq = rq;
  a.cp_min_bytes = rp.cp_min_bytes;
  a.cp_min_rows = rp.cp_min_rows;
  a.ids_local = ids_local;
  a.chunk_count = sel_local ? static_cast<const uint32_t *>(sel_scratch) : nullptr;
  CUDA_TRY(launch_range_count(a, gp, r, stream, &launches));
  int64_t C = 0;
  CUDA_TRY(cudaMemcpyAsync(&C, r.coff + (size_t)L * q, 8, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  Scratch scr2{ix->has_alloc ? &ix->alloc : nullptr, stream};
  st = scratch_alloc(scr2, carve_size({(size_t)C * 4, (size_t)C * 8, (size_t)C}));
  if (st != VRS_OK) return st;
  Carve cv2(scr2.ptr);
  r.cand = cv2.take<int32_t>((size_t)C);
  r.score = cv2.take<double>((size_t)C);
  r.keep = cv2.take<uint8_t>((size_t)C);
  CUDA_TRY(launch_range_fill(a, gp, r, stream, &launches));
  int64_t R = 0;
  CUDA_TRY(cudaMemcpyAsync(&R, offsets + q, 8, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  *total = R;
  g_last_path = VRS_PATH_GEMM;
  g_last_prec = use16 ? ix->prec16 : VRS_PREC_TF32;
  if (R > capacity) {
    g_last_launches = launches;
    return fail(VRS_ERANGE, "%lld results > capacity %lld", (long long)R, (long long)capacity);
  }
  CUDA_TRY(launch_range_write(a, gp, r, stream, &launches));
  g_last_launches = launches;
  return VRS_OK;
}

vrs_status vrs_search_host(vrs_index *ix, const float *h_queries, int64_t q, int32_t d,
                           const vrs_predicate *pred, int32_t k, vrs_metric metric, int64_t *h_ids,
                           float *h_dists, const vrs_search_options *opts, void *cuda_stream) {
  g_err[0] = 0;
  if (!ix) return fail(VRS_EINVAL, "index is NULL");
  if (q < 0 || k < 1) return fail(VRS_EINVAL, "q < 0 or k < 1");
  if (q == 0) return vrs_search_ex(ix, nullptr, 0, d, pred, k, metric, nullptr, nullptr, opts, cuda_stream);
  if (!h_queries || !h_ids || !h_dists) return fail(VRS_EINVAL, "NULL host buffer");
  if (d != ix->d) return fail(VRS_EINVAL, "d = %d differs from the loaded d = %d", d, ix->d);
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  std::lock_guard<std::mutex> guard(ix->host_mu);
  if (!ix->up_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ix->up_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&ix->down_stream, cudaStreamNonBlocking));
    for (int i = 0; i < vrs_index::kSlots; ++i) {
      CUDA_TRY(cudaEventCreateWithFlags(&ix->slot_free[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&ix->up_done[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&ix->comp_done[i], cudaEventDisableTiming));
    }
  }
  const int slot = ix->slot_next;
  ix->slot_next = (slot + 1) % vrs_index::kSlots;
  const size_t qb = (size_t)q * d * 4, ib = (size_t)q * k * 8, db = (size_t)q * k * 4;
  const size_t need = carve_size({qb, ib, db});
  if (ix->slot_cap[slot] < need) {
    // grow (rare): every slot at once, to the new largest size -- the slots take turns,
    // so growing one at a time would stall (sync + free + malloc) on several later calls
    for (int i = 0; i < vrs_index::kSlots; ++i) {
      CUDA_TRY(cudaEventSynchronize(ix->slot_free[i]));   // (never-recorded events are complete)
      slot_release(ix, i);
    }
    for (int i = 0; i < vrs_index::kSlots; ++i) {
      void *p = nullptr;
      if (ix->has_alloc) p = ix->alloc.alloc(need, nullptr, ix->alloc.ctx);   // (index-owned, stream-free use)
      else if (cudaMalloc(&p, need) != cudaSuccess) { cudaGetLastError(); p = nullptr; }
      if (!p) return fail(VRS_ENOMEM, "allocation of %zu bytes for the host-call staging failed", need);
      ix->slot_buf[i] = p;
      ix->slot_cap[i] = need;
    }
  }
  Carve cv(ix->slot_buf[slot]);
  float *dq = cv.take<float>((size_t)q * d);
  int64_t *di = cv.take<int64_t>((size_t)q * k);
  float *dd = cv.take<float>((size_t)q * k);
  // upload (its own stream, once the slot's previous results are downloaded)
  CUDA_TRY(cudaStreamWaitEvent(ix->up_stream, ix->slot_free[slot], 0));
  CUDA_TRY(cudaMemcpyAsync(dq, h_queries, qb, cudaMemcpyHostToDevice, ix->up_stream));
  CUDA_TRY(cudaEventRecord(ix->up_done[slot], ix->up_stream));
  // search on the caller's stream
  CUDA_TRY(cudaStreamWaitEvent(stream, ix->up_done[slot], 0));
  vrs_status st = vrs_search_ex(ix, dq, q, d, pred, k, metric, di, dd, opts, cuda_stream);
  if (st != VRS_OK) return st;
  CUDA_TRY(cudaEventRecord(ix->comp_done[slot], stream));
  // download (its own stream), then the caller's stream waits for it so that
  // synchronising the caller's stream covers the host results
  CUDA_TRY(cudaStreamWaitEvent(ix->down_stream, ix->comp_done[slot], 0));
  CUDA_TRY(cudaMemcpyAsync(h_ids, di, ib, cudaMemcpyDeviceToHost, ix->down_stream));
  CUDA_TRY(cudaMemcpyAsync(h_dists, dd, db, cudaMemcpyDeviceToHost, ix->down_stream));
  CUDA_TRY(cudaEventRecord(ix->slot_free[slot], ix->down_stream));
  ix->last_down = slot;
  const int mode = opts ? opts->host_async : 0;
  if (mode != 2) CUDA_TRY(cudaStreamWaitEvent(stream, ix->slot_free[slot], 0));
  if (mode == 0) CUDA_TRY(cudaStreamSynchronize(stream));
  return VRS_OK;
}

vrs_status vrs_host_fence(vrs_index *ix, void *cuda_stream) {
  g_err[0] = 0;
  if (!ix) return fail(VRS_EINVAL, "index is NULL");
  std::lock_guard<std::mutex> guard(ix->host_mu);
  // the download stream is in order: its last recorded event covers every earlier copy
  if (ix->down_stream && ix->last_down >= 0)
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)cuda_stream, ix->slot_free[ix->last_down], 0));
  return VRS_OK;
}

vrs_status vrs_select(vrs_index *ix, const vrs_predicate *pred, uint32_t *bitmap, int64_t *count, int32_t *ids,
                      void *cuda_stream) {
  g_err[0] = 0;
  if (!ix) return fail(VRS_EINVAL, "index is NULL");
  PredDev pd;
  vrs_status st = make_pred(ix, pred, &pd);
  if (st != VRS_OK) return st;
  if (!is_device_ptr(bitmap) || !is_device_ptr(count)) return fail(VRS_EINVAL, "bitmap / count must be device pointers");
  if (ids && !is_device_ptr(ids)) return fail(VRS_EINVAL, "ids must be a device pointer");
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  Scratch scr{ix->has_alloc ? &ix->alloc : nullptr, stream};
  st = scratch_alloc(scr, select_scratch_bytes(ix->n));
  if (st != VRS_OK) return st;
  int launches = 0;
  CUDA_TRY(launch_select(pd, ix->n, bitmap, ids, count, scr.ptr, stream, &launches));
  g_last_launches = launches;
  return VRS_OK;
}

vrs_status vrs_merge(const int64_t *cand_ids, const float *cand_dists, int32_t n_parts, int64_t q, int32_t k,
                     vrs_metric metric, int64_t *ids, float *dists, void *cuda_stream) {
  g_err[0] = 0;
  if (n_parts < 1 || q < 0 || k < 1) return fail(VRS_EINVAL, "n_parts < 1, q < 0 or k < 1");
  if (metric != VRS_L2 && metric != VRS_IP && metric != VRS_COSINE)
    return fail(VRS_EINVAL, "bad metric %d", (int)metric);
  if (k > VRS_K_MAX) return fail(VRS_EUNSUPPORTED, "k = %d > VRS_K_MAX (%d)", k, VRS_K_MAX);
  if (q == 0) return VRS_OK;
  if (!is_device_ptr(cand_ids) || !is_device_ptr(cand_dists) || !is_device_ptr(ids) || !is_device_ptr(dists))
    return fail(VRS_EINVAL, "vrs_merge buffers must be device pointers");
  vrs_status st = check_device(nullptr, nullptr);
  if (st != VRS_OK) return st;
  int launches = 0;
  MergeArgs a{cand_ids, cand_dists, n_parts, q, k, (int32_t)metric, ids, dists};
  {
    ProfScope ps("merge", (cudaStream_t)cuda_stream);
    CUDA_TRY(launch_merge(a, (cudaStream_t)cuda_stream, &launches));
  }
  g_last_launches = launches;
  return VRS_OK;
}

vrs_status vrs_merge_push(const int64_t *local_ids, const float *local_dists, void *const *peer_bufs,
                          int64_t buf_bytes, int32_t n_parts, int32_t my_part, int64_t q, int32_t k,
                          vrs_metric metric, uint32_t *state, int64_t *ids, float *dists, void *cuda_stream) {
  g_err[0] = 0;
  if (n_parts < 1 || my_part < 0 || my_part >= n_parts || q < 0 || k < 1)
    return fail(VRS_EINVAL, "n_parts %d, my_part %d, q %lld, k %d", n_parts, my_part, (long long)q, k);
  if (n_parts > kPushMaxParts) return fail(VRS_EUNSUPPORTED, "n_parts = %d > %d", n_parts, kPushMaxParts);
  if (metric != VRS_L2 && metric != VRS_IP && metric != VRS_COSINE)
    return fail(VRS_EINVAL, "bad metric %d", (int)metric);
  if (k > VRS_K_MAX) return fail(VRS_EUNSUPPORTED, "k = %d > VRS_K_MAX (%d)", k, VRS_K_MAX);
  if (q == 0) return VRS_OK;
  if (buf_bytes < push_buffer_bytes(n_parts, q, k))
    return fail(VRS_EINVAL, "receive buffers of %lld bytes < %lld needed", (long long)buf_bytes,
                (long long)push_buffer_bytes(n_parts, q, k));
  if (!is_device_ptr(local_ids) || !is_device_ptr(local_dists) || !is_device_ptr(peer_bufs) || !is_device_ptr(state) ||
      !is_device_ptr(ids) || !is_device_ptr(dists))
    return fail(VRS_EINVAL, "vrs_merge_push buffers must be device pointers");
  vrs_status st = check_device(nullptr, nullptr);
  if (st != VRS_OK) return st;
  int launches = 0;
  // bound of the device-side wait for the peers' pushes (default 20 s; state[3] is set when it expires)
  static const long wait_ms = getenv("VRS_PUSH_TIMEOUT_MS") ? atol(getenv("VRS_PUSH_TIMEOUT_MS")) : 20000;
  PushMergeArgs a{local_ids, local_dists, peer_bufs, n_parts, my_part, q, k, (int32_t)metric, state, ids, dists,
                  (uint64_t)(wait_ms > 0 ? wait_ms : 1) * 1000000ull};
  {
    ProfScope ps("merge", (cudaStream_t)cuda_stream);
    CUDA_TRY(launch_push_merge(a, (cudaStream_t)cuda_stream, &launches));
  }
  g_last_launches = launches;
  return VRS_OK;
}

int64_t vrs_push_buffer_bytes(int32_t n_parts, int64_t q, int32_t k) { return push_buffer_bytes(n_parts, q, k); }

}  // extern "C"

#ifdef VRS_TC_TIMING
// Debug builds only (-DVRS_TC_TIMING): per-CTA timeline stamps of one translation
// unit's kernels (0 select.cu, 1 gemm_tc.cu, 2 finalize.cu; [8][4096][8] u64, see
// TL_STAMP in vrs_internal.cuh) copied to host and cleared.
namespace vrs {
int tl_read_select(unsigned long long *);
int tl_read_gemm(unsigned long long *);
int tl_read_fin(unsigned long long *);
}
extern "C" VRS_API int vrs_debug_timeline(int tu, unsigned long long *host) {
  return tu == 0 ? vrs::tl_read_select(host) : tu == 1 ? vrs::tl_read_gemm(host) : tu == 2 ? vrs::tl_read_fin(host) : -1;
}
#endif
