// C-ABI entry points of libtsketch (include/tsketch.h): argument validation, host/device
// pointer handling, and composition of the kernels into the calls of Algorithm 2
// (PAPER.md:156-169).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL itself is dlopen'ed (nccl_api below)

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>

#include "tsk_internal.h"

using tsk::Ctx;

namespace {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

tsk_status cuda_ok(cudaError_t e) {
  if (e == cudaSuccess) return TSK_OK;
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? TSK_ENOMEM : TSK_ECUDA;
}

bool is_error(tsk_status s) { return (int)s < 0; }

// device fp32 matrices are read with float4 / TMA: 16-byte alignment (host inputs are staged)
bool misaligned16(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

// Device view of a possibly-host buffer: allocated from a dedicated ctx workspace slot.
struct DevBuf {
  void* dev = nullptr;
  const void* user = nullptr;
  size_t bytes = 0;
  bool staged = false;
};

tsk_status stage_out(Ctx* c, DevBuf& b) {
  if (!b.staged || !b.user) return TSK_OK;
  tsk_status s = cuda_ok(cudaMemcpyAsync(const_cast<void*>(b.user), b.dev, b.bytes, cudaMemcpyDeviceToHost, c->stream));
  if (is_error(s)) return s;
  return cuda_ok(cudaStreamSynchronize(c->stream));
}

}  // namespace

// ------------------------------------------------------------------- extended ctx (streams for e2e)
struct CtxExt {
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr};
  cudaEvent_t consumed[2] = {nullptr, nullptr};
  void* buf[2] = {nullptr, nullptr};
  size_t buf_bytes = 0;
  void* dev_small[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t dev_small_bytes[4] = {0, 0, 0, 0};
  cudaEvent_t handoff = nullptr;  // tsk_set_stream: the new stream waits for the old one
};

struct tsk_ctx_full {
  tsk_ctx_s base;
  CtxExt ext;
};

static CtxExt* ext_of(tsk_ctx ctx) { return &reinterpret_cast<tsk_ctx_full*>(ctx)->ext; }

static void* small_ws(tsk_ctx ctx, int slot, size_t bytes) {
  CtxExt* e = ext_of(ctx);
  if (e->dev_small_bytes[slot] >= bytes) return e->dev_small[slot];
  if (e->dev_small[slot]) {
    cudaStreamSynchronize(ctx->c.stream);
    cudaFree(e->dev_small[slot]);
  }
  e->dev_small[slot] = nullptr;
  e->dev_small_bytes[slot] = 0;
  if (cudaMalloc(&e->dev_small[slot], bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  e->dev_small_bytes[slot] = bytes;
  return e->dev_small[slot];
}

// stage through an ext slot (used for outputs / small inputs)
static tsk_status stage_slot(tsk_ctx ctx, const void* user, size_t bytes, int slot, DevBuf& out, bool copy_in) {
  out.user = user;
  out.bytes = bytes;
  if (is_device_ptr(user)) {
    out.dev = const_cast<void*>(user);
    out.staged = false;
    return TSK_OK;
  }
  out.dev = small_ws(ctx, slot, bytes);
  if (!out.dev) return TSK_ENOMEM;
  out.staged = true;
  if (copy_in) return cuda_ok(cudaMemcpyAsync(out.dev, user, bytes, cudaMemcpyHostToDevice, ctx->c.stream));
  return TSK_OK;
}

// ---------------------------------------------------------------- NCCL, loaded at run time
// (types from nccl.h; the library itself is dlopen'ed so libtsketch has no link-time NCCL dependency
// and shares the copy torch already loaded)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.allGather;
  });
  return api.ok ? &api : nullptr;
}

namespace tsk {
// G (+)= over all ranks of the ctx's communicator (in place, fp64 sum) on the ctx stream
tsk_status allreduce_gram(Ctx* c, double* G, size_t n) {
  if (!c->comm) return TSK_OK;
  NcclApi* api = nccl_api();
  if (!api) return TSK_ENCCL;
  if (api->allReduce(G, G, n, ncclFloat64, ncclSum, reinterpret_cast<ncclComm_t>(c->comm), c->stream) != ncclSuccess)
    return TSK_ENCCL;
  return TSK_OK;
}
// every rank learns the worst status of the pre-collective phase (ncclMin over int32: errors are
// negative), so a rank that fails before the Gram all-reduce cannot leave its peers blocked in it
tsk_status allreduce_status(Ctx* c, tsk_status local) {
  if (!c->comm) return local;
  NcclApi* api = nccl_api();
  if (!api) return TSK_ENCCL;
  int* d = reinterpret_cast<int*>(c->workspace(WS_CHECK, 64));
  int* h = reinterpret_cast<int*>(c->pinned(64));
  if (!d || !h) return TSK_ENOMEM;
  h[0] = (int)local;
  if (cudaMemcpyAsync(d, h, sizeof(int), cudaMemcpyHostToDevice, c->stream) != cudaSuccess) return TSK_ECUDA;
  if (api->allReduce(d, d, 1, ncclInt32, ncclMin, reinterpret_cast<ncclComm_t>(c->comm), c->stream) != ncclSuccess)
    return TSK_ENCCL;
  if (cudaMemcpyAsync(h, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return TSK_ECUDA;
  return (tsk_status)std::min(h[0], (int)local);
}
}  // namespace tsk

// out[b] = pad[rank(b)][b - lo(rank(b))]: compaction of the padded all-gather of contiguous shards
__global__ void unpad_gather_kernel(const double* __restrict__ pad, long long per, long long B, int P,
                                    double* __restrict__ out) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  // rank of index b under shard_range: the largest p with floor(p B / P) <= b
  long long p = (b * P) / B;
  while (p + 1 < P && ((p + 1) * B) / P <= b) ++p;
  while (p > 0 && (p * B) / P > b) --p;
  out[b] = pad[p * per + (b - (p * B) / P)];
}

// ------------------------------------------------------------------------------ whole-array staging
// Host pointers for the entry points that consume whole arrays (two-sided, matrix-free): every host
// buffer gets a device copy in a ctx staging slot (inputs copied in on the ctx stream, outputs copied
// back), and the call returns after the stream is synchronised -- the synchronous host semantics of the
// one-sided entry points (which additionally chunk A through pinned double buffers).  Device buffers are
// used in place and must be 16-byte aligned (TMA rows).
namespace {
struct Stager {
  tsk::Ctx* c;
  int next = tsk::WS_STAGE_0;
  tsk_status st = TSK_OK;
  bool any = false;
  struct Out {
    void* dev;
    void* user;
    size_t bytes;
  };
  Out outs[8];
  int nout = 0;
  void* slot(size_t bytes) {
    if (next > tsk::WS_STAGE_LAST) {
      st = TSK_EINVAL;
      return nullptr;
    }
    void* d = c->workspace(next++, bytes);
    if (!d) st = TSK_ENOMEM;
    any = true;
    return d;
  }
  template <class T>
  const T* in(const T* user, size_t bytes) {
    if (!user || st != TSK_OK) return user;
    if (is_device_ptr(user)) {
      if (misaligned16(user)) st = TSK_ESHAPE;
      return user;
    }
    void* d = slot(bytes);
    if (d && cudaMemcpyAsync(d, user, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) st = TSK_ECUDA;
    return reinterpret_cast<const T*>(d);
  }
  template <class T>
  T* out(T* user, size_t bytes) {
    if (!user || st != TSK_OK) return user;
    if (is_device_ptr(user)) {
      if (misaligned16(user) && sizeof(T) == 4) st = TSK_ESHAPE;
      return user;
    }
    void* d = slot(bytes);
    if (d) outs[nout++] = Out{d, user, bytes};
    return reinterpret_cast<T*>(d);
  }
  // copy the outputs back (also after a warning status) and synchronise when anything was staged
  tsk_status finish(tsk_status s) {
    if (is_error(s)) {
      if (any) cudaStreamSynchronize(c->stream);
      return s;
    }
    for (int i = 0; i < nout; ++i)
      if (cudaMemcpyAsync(outs[i].user, outs[i].dev, outs[i].bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
        return TSK_ECUDA;
    if (any && cudaStreamSynchronize(c->stream) != cudaSuccess) return TSK_ECUDA;
    return s;
  }
};
}  // namespace

extern "C" {

tsk_status tsk_get_unique_id(unsigned char uid[128]) {
  if (!uid) return TSK_ENULL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  NcclApi* api = nccl_api();
  if (!api) return TSK_ENCCL;
  ncclUniqueId id;
  if (api->getUniqueId(&id) != ncclSuccess) return TSK_ENCCL;
  memcpy(uid, &id, sizeof(id));
  return TSK_OK;
}

tsk_status tsk_comm_init(tsk_ctx ctx, int nranks, int rank, const unsigned char uid[128]) {
  if (!ctx || !uid) return TSK_ENULL;
  if (nranks < 1 || rank < 0 || rank >= nranks) return TSK_EINVAL;
  NcclApi* api = nccl_api();
  if (!api) return TSK_ENCCL;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  if (c.comm) {
    cudaStreamSynchronize(c.stream);
    api->commDestroy(reinterpret_cast<ncclComm_t>(c.comm));
    c.comm = nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  if (api->commInitRank(&comm, nranks, id, rank) != ncclSuccess) return TSK_ENCCL;
  c.comm = comm;
  c.nranks = nranks;
  c.rank = rank;
  return TSK_OK;
}

tsk_status tsk_allreduce_gram(tsk_ctx ctx, double* G64, int m) {
  if (!ctx) return TSK_ENULL;
  if (!G64) return TSK_ENULL;
  if (m < 1) return TSK_EINVAL;
  if (!is_device_ptr(G64)) return TSK_EINVAL;
  cudaSetDevice(ctx->c.device);
  return tsk::allreduce_gram(&ctx->c, G64, (size_t)m * m);
}

tsk_status tsk_allgather_errors(tsk_ctx ctx, const double* err_local, int64_t B_total, double* err_all) {
  if (!ctx) return TSK_ENULL;
  if (B_total < 0) return TSK_EINVAL;
  Ctx& c = ctx->c;
  const int P = c.comm ? c.nranks : 1, rank = c.comm ? c.rank : 0;
  const int64_t lo = (int64_t)rank * B_total / P, hi = (int64_t)(rank + 1) * B_total / P;
  if (B_total == 0) return TSK_OK;
  if (!err_all || (hi > lo && !err_local)) return TSK_ENULL;
  if (!is_device_ptr(err_all) || (hi > lo && !is_device_ptr(err_local))) return TSK_EINVAL;
  cudaSetDevice(c.device);
  if (!c.comm)
    return cuda_ok(cudaMemcpyAsync(err_all, err_local, (size_t)B_total * 8, cudaMemcpyDeviceToDevice, c.stream));
  NcclApi* api = nccl_api();
  if (!api) return TSK_ENCCL;
  // shards differ by at most one: pad to the largest, gather [P][per], compact in shard order
  const int64_t per = (B_total + P - 1) / P;
  double* pad = reinterpret_cast<double*>(c.workspace(tsk::WS_GATHER, (size_t)(P + 1) * per * 8));
  if (!pad) return TSK_ENOMEM;
  double* mine = pad + (size_t)P * per;
  if (cudaMemsetAsync(mine, 0, (size_t)per * 8, c.stream) != cudaSuccess) return TSK_ECUDA;
  if (hi > lo && cudaMemcpyAsync(mine, err_local, (size_t)(hi - lo) * 8, cudaMemcpyDeviceToDevice, c.stream) !=
                     cudaSuccess)
    return TSK_ECUDA;
  if (api->allGather(mine, pad, (size_t)per, ncclFloat64, reinterpret_cast<ncclComm_t>(c.comm), c.stream) !=
      ncclSuccess)
    return TSK_ENCCL;
  unpad_gather_kernel<<<(unsigned)((B_total + 255) / 256), 256, 0, c.stream>>>(pad, per, B_total, P, err_all);
  c.count_launch();
  return tsk::launch_status("tsk_allgather_errors");
}

const char* tsk_status_string(tsk_status s) {
  switch (s) {
    case TSK_OK: return "ok";
    case TSK_WARN_RANK_CLAMPED: return "warning: r clamped to k";
    case TSK_WARN_NOT_CONVERGED: return "warning: eigensolver reached max_iters";
    case TSK_EINVAL: return "invalid argument";
    case TSK_ESHAPE: return "unsupported shape / alignment (n % 4 != 0 or misaligned pointer)";
    case TSK_ENOMEM: return "device allocation failed";
    case TSK_ECUDA: return "CUDA error";
    case TSK_ENCCL: return "NCCL unavailable or NCCL call failed";
    case TSK_ENONFINITE: return "non-finite (NaN/Inf) entry in the training input";
    case TSK_EDEVICE: return "device is not sm_100 (B200)";
    case TSK_ENULL: return "required pointer is NULL";
    case TSK_ENUMERIC: return "numerical breakdown the fallbacks could not repair";
  }
  return "unknown status";
}

tsk_status tsk_create(tsk_ctx* out, int device, void* cuda_stream) {
  if (!out) return TSK_ENULL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return TSK_EDEVICE;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return TSK_ECUDA;
  if (prop.major != 10 || prop.minor != 0) return TSK_EDEVICE;
  if (cudaSetDevice(device) != cudaSuccess) return TSK_ECUDA;
  auto* full = new (std::nothrow) tsk_ctx_full();
  if (!full) return TSK_ENOMEM;
  full->base.c.device = device;
  full->base.c.num_sms = prop.multiProcessorCount;
  full->base.c.stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  *out = &full->base;
  return TSK_OK;
}

tsk_status tsk_destroy(tsk_ctx ctx) {
  if (!ctx) return TSK_ENULL;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  for (int i = 0; i < tsk::WS_COUNT; ++i)
    if (c.ws[i]) cudaFree(c.ws[i]);
  if (c.host_pinned) cudaFreeHost(c.host_pinned);
  if (c.comm) {
    if (NcclApi* api = nccl_api()) api->commDestroy(reinterpret_cast<ncclComm_t>(c.comm));
    c.comm = nullptr;
  }
  for (auto& st : c.side)
    if (st) cudaStreamDestroy(st);
  for (auto& ev : c.ev)
    if (ev) cudaEventDestroy(ev);
  CtxExt* e = ext_of(ctx);
  for (int i = 0; i < 2; ++i) {
    if (e->buf[i]) cudaFree(e->buf[i]);
    if (e->copied[i]) cudaEventDestroy(e->copied[i]);
    if (e->consumed[i]) cudaEventDestroy(e->consumed[i]);
  }
  for (int i = 0; i < 4; ++i)
    if (e->dev_small[i]) cudaFree(e->dev_small[i]);
  if (e->copy) cudaStreamDestroy(e->copy);
  if (e->handoff) cudaEventDestroy(e->handoff);
  delete reinterpret_cast<tsk_ctx_full*>(ctx);
  return TSK_OK;
}

tsk_status tsk_set_scw_error_mode(tsk_ctx ctx, int mode, double tau) {
  if (!ctx) return TSK_ENULL;
  if (mode < 0 || mode > 1 || !(tau < 1.0) || tau != tau) return TSK_EINVAL;
  ctx->c.scw_err_mode = mode;
  ctx->c.scw_tau = tau > 0.0 ? tau : 0.0;
  return TSK_OK;
}

tsk_status tsk_set_stream(tsk_ctx ctx, void* cuda_stream) {
  if (!ctx) return TSK_ENULL;
  Ctx& c = ctx->c;
  cudaStream_t ns = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (ns == c.stream) return TSK_OK;
  // work still queued on the old stream uses this ctx's workspaces: the new stream waits for it
  cudaSetDevice(c.device);
  CtxExt* e = ext_of(ctx);
  if (!e->handoff && cudaEventCreateWithFlags(&e->handoff, cudaEventDisableTiming) != cudaSuccess) return TSK_ECUDA;
  if (cudaEventRecord(e->handoff, c.stream) != cudaSuccess || cudaStreamWaitEvent(ns, e->handoff, 0) != cudaSuccess)
    return TSK_ECUDA;
  c.stream = ns;
  return TSK_OK;
}

tsk_status tsk_sync(tsk_ctx ctx) {
  if (!ctx) return TSK_ENULL;
  return cuda_ok(cudaStreamSynchronize(ctx->c.stream));
}

int64_t tsk_launch_count(tsk_ctx ctx) { return ctx ? ctx->c.launches : -1; }

// ------------------------------------------------------------------------------ training
// any NaN / Inf among n4 float4 (exponent field all ones); the order of the flag updates is irrelevant
__global__ void nonfinite_kernel(const float4* __restrict__ x, long long n4, int* __restrict__ flag) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    bad |= ((__float_as_uint(v.x) & 0x7F800000u) == 0x7F800000u) | ((__float_as_uint(v.y) & 0x7F800000u) == 0x7F800000u) |
           ((__float_as_uint(v.z) & 0x7F800000u) == 0x7F800000u) | ((__float_as_uint(v.w) & 0x7F800000u) == 0x7F800000u);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static tsk_status check_finite(Ctx* c, const float* A, long long count) {
  int* flag = reinterpret_cast<int*>(c->workspace(tsk::WS_CHECK, 64));
  int* hflag = reinterpret_cast<int*>(c->pinned(64));
  if (!flag || !hflag) return TSK_ENOMEM;
  if (cudaMemsetAsync(flag, 0, sizeof(int), c->stream) != cudaSuccess) return TSK_ECUDA;
  nonfinite_kernel<<<4 * c->num_sms, 256, 0, c->stream>>>(reinterpret_cast<const float4*>(A), count / 4, flag);
  c->count_launch();
  if (cudaMemcpyAsync(hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return TSK_ECUDA;
  return *hflag ? TSK_ENONFINITE : TSK_OK;
}

static tsk_status gram_device(Ctx* c, const float* A, int64_t D, int m, int n, double* G64, float* G32,
                              int accumulate, const tsk_train_opts* opts, tsk_train_info* info) {
  if (opts && opts->check_finite) {
    const tsk_status fs = check_finite(c, A, (long long)D * m * n);  // n % 4 == 0: whole float4s
    if (fs != TSK_OK) return fs;
  }
  tsk::GemmProblem p;
  p.X = A;
  p.Y = A;
  p.M = m;
  p.N = m;
  p.n = n;
  p.D = D;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.y_row_stride = n;
  p.y_slice_stride = (long long)m * n;
  p.sym = 1;
  p.out64 = G64;
  p.ldo64 = m;
  p.out32 = G32;
  p.ldo32 = m;
  p.accumulate = accumulate;
  if (opts) {
    p.chain = opts->gemm_chain;
    p.splits = opts->gemm_splits;
  }
  tsk::GemmInfo gi;
  p.info = &gi;
  tsk_status s = tsk::gemm_tf32x3(c, p);
  if (info && s == TSK_OK) {
    info->gram_splits = gi.splits;
    info->gram_tiles = gi.tiles;
  }
  return s;
}

// Host-resident training stack: stream it through two device buffers, overlapping the
// H2D copy of chunk i+1 with the Gram of chunk i (accumulating into G64).
static tsk_status gram_host(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, float* G32,
                            int accumulate, const tsk_train_opts* opts, tsk_train_info* info) {
  Ctx* c = &ctx->c;
  CtxExt* e = ext_of(ctx);
  const size_t mat = (size_t)m * n * 4;
  const size_t target = (size_t)256 << 20;  // 256 MiB per staging buffer
  int64_t chunk = std::max<int64_t>(1, (int64_t)(target / mat));
  chunk = std::min<int64_t>(chunk, D);
  const size_t bytes = (size_t)chunk * mat;
  if (!e->copy) {
    if (cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking) != cudaSuccess) return TSK_ECUDA;
    for (int i = 0; i < 2; ++i) {
      cudaEventCreateWithFlags(&e->copied[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&e->consumed[i], cudaEventDisableTiming);
    }
  }
  if (e->buf_bytes < bytes) {
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < 2; ++i) {
      if (e->buf[i]) cudaFree(e->buf[i]);
      e->buf[i] = nullptr;
      if (cudaMalloc(&e->buf[i], bytes) != cudaSuccess) {
        cudaGetLastError();
        e->buf_bytes = 0;
        return TSK_ENOMEM;
      }
    }
    e->buf_bytes = bytes;
  }
  // the copy stream must not start before earlier work on the compute stream released the buffers
  cudaEventRecord(e->consumed[0], c->stream);
  cudaEventRecord(e->consumed[1], c->stream);
  int i = 0;
  for (int64_t d0 = 0; d0 < D; d0 += chunk, i ^= 1) {
    const int64_t dc = std::min<int64_t>(chunk, D - d0);
    cudaStreamWaitEvent(e->copy, e->consumed[i], 0);
    if (cudaMemcpyAsync(e->buf[i], A + (size_t)d0 * m * n, (size_t)dc * mat, cudaMemcpyHostToDevice, e->copy) !=
        cudaSuccess)
      return TSK_ECUDA;
    cudaEventRecord(e->copied[i], e->copy);
    cudaStreamWaitEvent(c->stream, e->copied[i], 0);
    const bool last = d0 + dc >= D;
    tsk_status s = gram_device(c, reinterpret_cast<const float*>(e->buf[i]), dc, m, n, G64, last ? G32 : nullptr,
                               (d0 == 0) ? accumulate : 1, opts, info);
    if (is_error(s)) return s;
    cudaEventRecord(e->consumed[i], c->stream);
  }
  // host inputs are synchronous (include/tsketch.h): the caller may refill its buffer on return
  return cuda_ok(cudaStreamSynchronize(c->stream));
}

tsk_status sketch_gram(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, float* G32, int accumulate,
                       const tsk_train_opts* opts, tsk_train_info* info) {
  if (!ctx) return TSK_ENULL;
  if (!A || !G64) return TSK_ENULL;
  if (D < 1 || m < 1 || n < 1) return TSK_EINVAL;
  if (n % 4) return TSK_ESHAPE;
  if (is_device_ptr(A) && misaligned16(A)) return TSK_ESHAPE;
  Ctx* c = &ctx->c;
  cudaSetDevice(c->device);
  DevBuf g64, g32;
  tsk_status s = stage_slot(ctx, G64, (size_t)m * m * 8, 0, g64, accumulate != 0);
  if (is_error(s)) return s;
  if (G32) {
    s = stage_slot(ctx, G32, (size_t)m * m * 4, 1, g32, false);
    if (is_error(s)) return s;
  }
  float* g32d = G32 ? reinterpret_cast<float*>(g32.dev) : nullptr;
  if (is_device_ptr(A))
    s = gram_device(c, A, D, m, n, reinterpret_cast<double*>(g64.dev), g32d, accumulate, opts, info);
  else
    s = gram_host(ctx, A, D, m, n, reinterpret_cast<double*>(g64.dev), g32d, accumulate, opts, info);
  if (is_error(s)) return s;
  if (g64.staged) {
    if (is_error(s = stage_out(&ctx->c, g64))) return s;
  }
  if (G32 && g32.staged) {
    if (is_error(s = stage_out(&ctx->c, g32))) return s;
  }
  return TSK_OK;
}

// the eigensolver's Rayleigh-Ritz block p = min(m, k + oversample) must be <= 128 above the dense path
static bool block_ok(int m, int k, const tsk_train_opts* opts) {
  const int dense = opts && opts->dense_max_m > 0 ? std::min(opts->dense_max_m, 256) : 256;
  const int q = opts && opts->oversample > 0 ? opts->oversample : 16;
  const int p = std::min(m, k + q);
  return m <= dense || p >= m ? m <= 256 : p <= 128;
}

tsk_status sketch_topk(tsk_ctx ctx, const double* G64, int m, int k, float* S, double* lambda,
                       const tsk_train_opts* opts, tsk_train_info* info) {
  if (!ctx) return TSK_ENULL;
  if (!G64 || !S) return TSK_ENULL;
  if (m < 1 || k < 1 || k > m) return TSK_EINVAL;
  if (!block_ok(m, k, opts)) return TSK_EINVAL;
  cudaSetDevice(ctx->c.device);
  DevBuf g, sb, lb;
  tsk_status s = stage_slot(ctx, G64, (size_t)m * m * 8, 0, g, true);
  if (is_error(s)) return s;
  if (is_error(s = stage_slot(ctx, S, (size_t)k * m * 4, 2, sb, false))) return s;
  if (lambda && is_error(s = stage_slot(ctx, lambda, (size_t)k * 8, 3, lb, false))) return s;
  tsk_status r = tsk::topk_eigen(&ctx->c, reinterpret_cast<const double*>(g.dev), m, k,
                                 reinterpret_cast<float*>(sb.dev), lambda ? reinterpret_cast<double*>(lb.dev) : nullptr,
                                 opts, info);
  if (is_error(r)) return r;
  if (is_error(s = stage_out(&ctx->c, sb))) return s;
  if (lambda && is_error(s = stage_out(&ctx->c, lb))) return s;
  return r;
}

tsk_status sketch_train(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, float* S, double* lambda,
                        double* G64_out, const tsk_train_opts* opts, tsk_train_info* info) {
  if (!ctx) return TSK_ENULL;
  Ctx* c = &ctx->c;
  cudaSetDevice(c->device);
  // Validation and the local Gram must not return early on a multi-rank communicator: every rank
  // joins the status all-reduce (below) so a failing rank cannot leave its peers in the Gram
  // all-reduce.  With a communicator a rank may own no training matrix (D = 0: zero contribution).
  tsk_status pre = TSK_OK;
  if (!S || (D > 0 && !A)) pre = TSK_ENULL;
  else if (D < (c->comm ? 0 : 1) || m < 1 || n < 1 || k < 1 || k > m || !block_ok(m, k, opts)) pre = TSK_EINVAL;
  else if (n % 4 || (D > 0 && is_device_ptr(A) && misaligned16(A))) pre = TSK_ESHAPE;
  double* G = nullptr;
  const bool g_dev = G64_out && is_device_ptr(G64_out);
  if (pre == TSK_OK) {
    if (g_dev) {
      G = G64_out;
    } else {
      G = reinterpret_cast<double*>(c->workspace(tsk::WS_GRAM, (size_t)m * m * 8));
      if (!G) pre = TSK_ENOMEM;
    }
  }
  if (pre == TSK_OK) {
    if (D == 0)
      pre = cuda_ok(cudaMemsetAsync(G, 0, (size_t)m * m * 8, c->stream));
    else if (is_device_ptr(A))
      pre = gram_device(c, A, D, m, n, G, nullptr, 0, opts, info);
    else
      pre = gram_host(ctx, A, D, m, n, G, nullptr, 0, opts, info);
  }
  tsk_status s = tsk::allreduce_status(c, pre);
  if (is_error(s)) return s;
  if (is_error(s = tsk::allreduce_gram(c, G, (size_t)m * m))) return s;  // multi-GPU (tsk_comm_init)
  DevBuf sb, lb;
  if (is_error(s = stage_slot(ctx, S, (size_t)k * m * 4, 2, sb, false))) return s;
  if (lambda && is_error(s = stage_slot(ctx, lambda, (size_t)k * 8, 3, lb, false))) return s;
  tsk_status r = tsk::topk_eigen(c, G, m, k, reinterpret_cast<float*>(sb.dev),
                                 lambda ? reinterpret_cast<double*>(lb.dev) : nullptr, opts, info);
  if (is_error(r)) return r;
  if (is_error(s = stage_out(&ctx->c, sb))) return s;
  if (lambda && is_error(s = stage_out(&ctx->c, lb))) return s;
  if (G64_out && !g_dev) {
    if (is_error(s = cuda_ok(cudaMemcpyAsync(G64_out, G, (size_t)m * m * 8, cudaMemcpyDeviceToHost, c->stream))))
      return s;
    if (is_error(s = cuda_ok(cudaStreamSynchronize(c->stream)))) return s;
  }
  return r;
}

// ------------------------------------------------------------------------------ test stream
static tsk_status scw_common(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k, int r,
                             float* L, float* R, float* sigma, double* err) {
  if (!ctx) return TSK_ENULL;
  if (B < 0 || m < 1 || n < 1 || k < 1 || k > m || r < 1) return TSK_EINVAL;
  if (B > 0 && (!A || !S)) return TSK_ENULL;
  if (n % 4) return TSK_ESHAPE;
  if (B > 0 && is_device_ptr(A) && misaligned16(A)) return TSK_ESHAPE;
  if (k > 128) return TSK_EINVAL;
  tsk_status warn = TSK_OK;
  if (r > k) {
    r = k;
    warn = TSK_WARN_RANK_CLAMPED;
  }
  if (r > std::min(m, n) || r > 64) return TSK_EINVAL;
  if (B == 0) return warn;
  Ctx* c = &ctx->c;
  cudaSetDevice(c->device);
  DevBuf sb;
  tsk_status s = stage_slot(ctx, S, (size_t)k * m * 4, 2, sb, true);
  if (is_error(s)) return s;
  const float* Sd = reinterpret_cast<const float*>(sb.dev);
  const bool a_dev = is_device_ptr(A);
  const bool out_dev = (!L || is_device_ptr(L)) && (!R || is_device_ptr(R)) && (!sigma || is_device_ptr(sigma)) &&
                       (!err || is_device_ptr(err));
  if (a_dev && out_dev) {
    s = tsk::scw_run(c, A, B, m, n, Sd, k, r, L, R, sigma, err);
    return is_error(s) ? s : warn;
  }
  // host path: chunk over matrices, stage in / run / copy results out
  const size_t mat = (size_t)m * n * 4;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(((size_t)512 << 20) / mat));
  chunk = std::min<int64_t>(chunk, B);
  float* Ad = nullptr;
  if (!a_dev) {
    Ad = reinterpret_cast<float*>(c->workspace(tsk::WS_HOST_IN, (size_t)chunk * mat));
    if (!Ad) return TSK_ENOMEM;
  }
  // staging for host outputs, sized with the same 256-byte rounding carve() applies per array
  auto r256 = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t out_bytes = (L ? r256((size_t)chunk * m * r * 4) : 0) + (R ? r256((size_t)chunk * n * r * 4) : 0) +
                           (sigma ? r256((size_t)chunk * r * 4) : 0) + (err ? r256((size_t)chunk * 8) : 0) + 256;
  uint8_t* Od = reinterpret_cast<uint8_t*>(c->workspace(tsk::WS_HOST_OUT, out_bytes));
  if (!Od) return TSK_ENOMEM;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t bc = std::min<int64_t>(chunk, B - b0);
    const float* Ac = A + (size_t)b0 * m * n;
    if (!a_dev) {
      if (is_error(s = cuda_ok(cudaMemcpyAsync(Ad, Ac, (size_t)bc * mat, cudaMemcpyHostToDevice, c->stream)))) return s;
      Ac = Ad;
    }
    uint8_t* o = Od;
    auto carve = [&](size_t bytes) {
      uint8_t* p = o;
      o += (bytes + 255) & ~size_t(255);
      return p;
    };
    float* Lc = L ? (is_device_ptr(L) ? L + (size_t)b0 * m * r : reinterpret_cast<float*>(carve((size_t)bc * m * r * 4))) : nullptr;
    float* Rc = R ? (is_device_ptr(R) ? R + (size_t)b0 * n * r : reinterpret_cast<float*>(carve((size_t)bc * n * r * 4))) : nullptr;
    float* sc = sigma ? (is_device_ptr(sigma) ? sigma + (size_t)b0 * r : reinterpret_cast<float*>(carve((size_t)bc * r * 4))) : nullptr;
    double* ec = err ? (is_device_ptr(err) ? err + b0 : reinterpret_cast<double*>(carve((size_t)bc * 8))) : nullptr;
    if (is_error(s = tsk::scw_run(c, Ac, bc, m, n, Sd, k, r, Lc, Rc, sc, ec))) return s;
    if (L && !is_device_ptr(L))
      cudaMemcpyAsync(L + (size_t)b0 * m * r, Lc, (size_t)bc * m * r * 4, cudaMemcpyDeviceToHost, c->stream);
    if (R && !is_device_ptr(R))
      cudaMemcpyAsync(R + (size_t)b0 * n * r, Rc, (size_t)bc * n * r * 4, cudaMemcpyDeviceToHost, c->stream);
    if (sigma && !is_device_ptr(sigma))
      cudaMemcpyAsync(sigma + (size_t)b0 * r, sc, (size_t)bc * r * 4, cudaMemcpyDeviceToHost, c->stream);
    if (err && !is_device_ptr(err)) cudaMemcpyAsync(err + b0, ec, (size_t)bc * 8, cudaMemcpyDeviceToHost, c->stream);
    if (is_error(s = cuda_ok(cudaStreamSynchronize(c->stream)))) return s;
  }
  return warn;
}

tsk_status sketch_apply_scw(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k, int r,
                            float* L, float* R, float* sigma) {
  return scw_common(ctx, A, B, m, n, S, k, r, L, R, sigma, nullptr);
}

tsk_status scw_error(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k, int r,
                     double* err) {
  if (!err && B > 0) return TSK_ENULL;
  return scw_common(ctx, A, B, m, n, S, k, r, nullptr, nullptr, nullptr, err);
}

// ------------------------------------------------------------------------------ two-sided variant
// (host or device pointers)
tsk_status sketch_gram_mode2(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, int accumulate) {
  if (!ctx) return TSK_ENULL;
  if (!A || !G64) return TSK_ENULL;
  if (D < 1 || m < 1 || n < 1) return TSK_EINVAL;
  if ((m % 4) || (n % 4)) return TSK_ESHAPE;
  cudaSetDevice(ctx->c.device);
  Stager sg{&ctx->c};
  const float* Ad = sg.in(A, (size_t)D * m * n * 4);
  double* Gd = accumulate ? const_cast<double*>(sg.in(G64, (size_t)n * n * 8)) : sg.out(G64, (size_t)n * n * 8);
  if (accumulate && Gd != G64 && sg.st == TSK_OK) sg.outs[sg.nout++] = Stager::Out{Gd, G64, (size_t)n * n * 8};
  if (sg.st != TSK_OK) return sg.finish(sg.st);
  return sg.finish(tsk::gram_mode2(&ctx->c, Ad, D, m, n, Gd, accumulate));
}

tsk_status sketch_train_two_sided(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, int l, float* S,
                                  float* W, const tsk_hooi_opts* opts, tsk_hooi_info* info) {
  if (!ctx) return TSK_ENULL;
  if (!A || !S || !W) return TSK_ENULL;
  if (D < 1 || m < 1 || n < 1 || k < 1 || k > m || l < 1 || l > n) return TSK_EINVAL;
  if ((m % 4) || (n % 4)) return TSK_ESHAPE;
  if ((m > 256 && k + 16 > 256) || (n > 256 && l + 16 > 256)) return TSK_EINVAL;
  cudaSetDevice(ctx->c.device);
  Stager sg{&ctx->c};
  const float* Ad = sg.in(A, (size_t)D * m * n * 4);
  float* Sd = sg.out(S, (size_t)k * m * 4);
  float* Wd = sg.out(W, (size_t)l * n * 4);
  if (sg.st != TSK_OK) return sg.finish(sg.st);
  return sg.finish(tsk::hooi_tucker2(&ctx->c, Ad, D, m, n, k, l, Sd, Wd, opts, info));
}

// ------------------------------------------------------------------------------ matrix-free sketch
// (host or device pointers)
tsk_status sketch_train_matrix_free(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, float* S,
                                    double* lambda, const tsk_mf_opts* opts, tsk_mf_info* info) {
  if (!ctx) return TSK_ENULL;
  if (!A || !S) return TSK_ENULL;
  if (D < 1 || m < 1 || n < 1 || k < 1 || k > m) return TSK_EINVAL;
  if (n % 4) return TSK_ESHAPE;
  cudaSetDevice(ctx->c.device);
  Stager sg{&ctx->c};
  const float* Ad = sg.in(A, (size_t)D * m * n * 4);
  float* Sd = sg.out(S, (size_t)k * m * 4);
  double* ld = sg.out(lambda, (size_t)k * 8);
  tsk_mf_opts o{};
  if (opts) o = *opts;
  if (o.omega) {  // the start block [m][p], p as matrix_free_sketch derives it
    int pp = k + (o.oversample > 0 ? o.oversample : 16);
    pp = std::min((pp + 3) & ~3, m);
    o.omega = sg.in(o.omega, (size_t)m * pp * 8);
  }
  if (sg.st != TSK_OK) return sg.finish(sg.st);
  return sg.finish(tsk::matrix_free_sketch(&ctx->c, Ad, D, m, n, k, Sd, ld, opts ? &o : nullptr, info));
}

static tsk_status scw2_common(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k,
                              const float* W, int l, int r, float* L, float* R, float* sigma, double* err) {
  if (!ctx) return TSK_ENULL;
  if (B < 0 || m < 1 || n < 1 || k < 1 || k > m || l < 1 || l > n || r < 1) return TSK_EINVAL;
  if (B > 0 && (!A || !S || !W)) return TSK_ENULL;
  if ((m % 4) || (n % 4)) return TSK_ESHAPE;
  if (k > 116 || l > 116) return TSK_EINVAL;
  tsk_status warn = TSK_OK;
  if (r > std::min(k, l)) {
    r = std::min(k, l);
    warn = TSK_WARN_RANK_CLAMPED;
  }
  if (r > std::min(m, n) || r > 64) return TSK_EINVAL;
  if (B == 0) return warn;
  cudaSetDevice(ctx->c.device);
  Stager sg{&ctx->c};
  const float* Ad = sg.in(A, (size_t)B * m * n * 4);
  const float* Sd = sg.in(S, (size_t)k * m * 4);
  const float* Wd = sg.in(W, (size_t)l * n * 4);
  float* Ld = sg.out(L, (size_t)B * m * r * 4);
  float* Rd = sg.out(R, (size_t)B * n * r * 4);
  float* sd = sg.out(sigma, (size_t)B * r * 4);
  double* ed = sg.out(err, (size_t)B * 8);
  if (sg.st != TSK_OK) return sg.finish(sg.st);
  tsk_status s = sg.finish(tsk::scw2_run(&ctx->c, Ad, B, m, n, Sd, k, Wd, l, r, Ld, Rd, sd, ed));
  return is_error(s) ? s : warn;
}

tsk_status sketch_apply_two_sided_scw(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k,
                                      const float* W, int l, int r, float* L, float* R, float* sigma) {
  return scw2_common(ctx, A, B, m, n, S, k, W, l, r, L, R, sigma, nullptr);
}

tsk_status two_sided_scw_error(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k,
                               const float* W, int l, int r, double* err) {
  if (B > 0 && !err) return TSK_ENULL;
  return scw2_common(ctx, A, B, m, n, S, k, W, l, r, nullptr, nullptr, nullptr, err);
}

tsk_status tsk_gram_probe(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, int mode, int chain,
                          int splits) {
  if (!ctx) return TSK_ENULL;
  if (!A || !G64) return TSK_ENULL;
  if (D < 1 || m < 1 || n < 1) return TSK_EINVAL;
  if (n % 4) return TSK_ESHAPE;
  if (!is_device_ptr(A) || !is_device_ptr(G64)) return TSK_EINVAL;
  tsk::GemmProblem p;
  p.X = A;
  p.Y = A;
  p.M = m;
  p.N = m;
  p.n = n;
  p.D = D;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.y_row_stride = n;
  p.y_slice_stride = (long long)m * n;
  p.sym = 1;
  p.out64 = G64;
  p.ldo64 = m;
  p.chain = chain;
  p.splits = splits;
  p.raw = mode & 1;
  p.products = (mode & 2) ? 1 : 3;
  p.lag = (mode & 4) ? 0 : -1;
  p.ss = (mode & 8) ? 1 : 0;
  p.one_cta = (mode & 16) ? 1 : 0;
  p.spin_waits = (mode & 32) ? 1 : 0;
  return tsk::gemm_tf32x3(&ctx->c, p);
}

tsk_status tsk_eig_probe(tsk_ctx ctx, const double* H, int p, int batch, double* W, double* lam, int* sweeps) {
  if (!ctx) return TSK_ENULL;
  if (!H || !W || !lam) return TSK_ENULL;
  if (p < 1 || p > 256 || batch < 0) return TSK_EINVAL;
  if (!is_device_ptr(H) || !is_device_ptr(W) || !is_device_ptr(lam) || (sweeps && !is_device_ptr(sweeps)))
    return TSK_EINVAL;
  return tsk::jacobi_eig_batched(&ctx->c, H, p, batch, W, lam, sweeps, 1e-13);
}

tsk_status tsk_syev_probe(tsk_ctx ctx, const double* H, int p, int nw, double* W, double* lam, int* flag,
                          double orth_tol) {
  if (!ctx) return TSK_ENULL;
  if (!H || !W || !lam) return TSK_ENULL;
  if (p < 1 || p > 256 || nw < 1 || nw > p) return TSK_EINVAL;
  if (!is_device_ptr(H) || !is_device_ptr(W) || !is_device_ptr(lam) || (flag && !is_device_ptr(flag)))
    return TSK_EINVAL;
  return tsk::syev_top(&ctx->c, H, p, nw, W, nw, lam, flag, orth_tol);
}

}  // extern "C"
