// Multi-GPU layer: one process per GPU, a symmetric device workspace mapped by
// every rank through CUDA IPC, device-side barriers on flag words in that
// workspace, and the three ZeRO++ collectives fused with their codec kernels
// over NVLink peer loads (no staging copies, no NCCL on the data path).
//
//   qwZ  zs/collectives.py:244-282   K0 -> world barrier -> K4 pulling peers' codes
//   hpZ  zs/collectives.py:202-241   (groups) group barrier -> peer copy of the
//                                    secondary shards held in HBM
//   qgZ  zs/collectives.py:464-569   per stage: K1 -> group barrier -> K2 pulling
//                                    the X intra messages -> cross barrier -> K3
//                                    pulling the Y hop-2 segments
//
// Double buffering: every use of a region alternates between two halves, and a
// rank only rewrites a half after passing a barrier that every reader of the
// previous contents must have reached after finishing its reads.
#include <cstring>
#include <vector>

#include "zpp_internal.h"
#include "zpp_kernels.cuh"
#include "zpp_launch.cuh"

using namespace zpp;

namespace {

constexpr int kMaxRanks = kMaxSrc;
constexpr int kScopes = 3;  // world, group, cross
constexpr size_t kFlagBytes = kScopes * kMaxRanks * sizeof(uint32_t);

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct BarrierArgs {
  uint32_t* remote[kMaxRanks];  // flag slot this rank writes in member m's buffer
  const uint32_t* local[kMaxRanks];  // flag slot member m writes in my buffer
};

__global__ void barrier_kernel(BarrierArgs a, int n, uint32_t epoch, uint64_t timeout_ns, uint32_t* flag) {
  if (comm_aborted(flag)) return;  // an earlier barrier timed out: stay stopped until the host resets
  const int t = threadIdx.x;
  __threadfence_system();
  __syncthreads();
  if (t < n) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.remote[t]), "r"(epoch) : "memory");
  }
  if (t < n) {
    const uint64_t t0 = globaltimer_ns();
    uint32_t v = 0;
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.local[t]) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        raise_flag(flag, FLAG_TIMEOUT);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

// byte copy of n_src peer segments into out (hpZ gather), 16 B vectors when aligned
__global__ void __launch_bounds__(256)
gather_copy_kernel(SrcTable src, int n_src, int rot, int64_t seg_bytes, uint8_t* __restrict__ out, int vec,
                   const uint32_t* flag) {
  if (comm_aborted(flag)) return;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (vec) {
    const int64_t units = seg_bytes / 16;
    const int64_t groups = (units + 31) / 32;
    for (int64_t g = gwarp; g < groups * n_src; g += nwarp) {
      const int s = (int)((g % n_src + rot) % n_src);
      const int64_t u = (g / n_src) * 32 + lane;
      if (u < units) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src.codes[s]) + u);
        reinterpret_cast<uint4*>(out + s * seg_bytes)[u] = v;
      }
    }
  } else {
    const int64_t total = seg_bytes * n_src;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int s = (int)(i / seg_bytes);
      out[i] = src.codes[s][i - s * seg_bytes];
    }
  }
}

// TMA-pipelined peer copy (hpZ gather): one elected thread streams 8 KB tiles
// of each group member's secondary shard into a 4-deep shared ring with
// cp.async.bulk; all threads write them out with 16-byte stores.
constexpr int kCopyStages = 4;
constexpr int kCopyTile = 8192;  // bytes

__global__ void __launch_bounds__(256)
gather_copy_tma_kernel(SrcTable src, int n_src, int rot, int64_t seg_bytes, uint8_t* __restrict__ out,
                       const uint32_t* flag) {
  if (comm_aborted(flag)) return;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* ring = dsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + kCopyStages * kCopyTile);
  const int tid = threadIdx.x;
  const int tiles = (int)((seg_bytes + kCopyTile - 1) / kCopyTile);
  const int n_tiles = tiles * n_src;
  if (tid == 0) {
    for (int i = 0; i < kCopyStages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto locate = [&](int g, int& s, int& t) {
    t = g / n_src;
    s = g - t * n_src + rot;
    if (s >= n_src) s -= n_src;
  };
  auto issue = [&](int g, int slot) {
    if (g < n_tiles) {
      int s, t;
      locate(g, s, t);
      const int64_t off = (int64_t)t * kCopyTile;
      const uint32_t bytes = (uint32_t)min((int64_t)kCopyTile, seg_bytes - off);
      mbar_expect_tx(&full[slot], bytes);
      bulk_g2s(ring + slot * kCopyTile, src.codes[s] + off, bytes, &full[slot]);
    }
  };
  const int G = gridDim.x;
  if (tid == 0)
    for (int k = 0; k < kCopyStages - 1; ++k) issue(blockIdx.x + k * G, k);
  int k = 0;
  for (int g = blockIdx.x; g < n_tiles; g += G, ++k) {
    const int slot = k % kCopyStages;
    if (tid == 0) issue(g + (kCopyStages - 1) * G, (k + kCopyStages - 1) % kCopyStages);
    mbar_wait(&full[slot], (uint32_t)((k / kCopyStages) & 1));
    int s, t;
    locate(g, s, t);
    const int64_t off = (int64_t)t * kCopyTile;
    const int bytes = (int)min((int64_t)kCopyTile, seg_bytes - off);
    uint8_t* dst = out + s * seg_bytes + off;
    const uint4* sm = reinterpret_cast<const uint4*>(ring + slot * kCopyTile);
    for (int i = tid; i < bytes / 16; i += 256) reinterpret_cast<uint4*>(dst)[i] = sm[i];
    __syncthreads();
  }
}

}  // namespace

static const int kTraceMax = 32;

struct zpp_comm {
  int rank = 0, world = 1, group = 1;
  size_t sym_bytes = 0;
  uint8_t* local = nullptr;        // this rank's symmetric buffer (sym_bytes + flags)
  uint8_t* peers[kMaxRanks] = {};  // every rank's buffer in this address space
  bool opened[kMaxRanks] = {};
  uint32_t epoch[kScopes] = {};
  uint64_t qwz_uses = 0, qgz_uses = 0;
  size_t qwz_region = 0;  // region size of the last qwZ call
  size_t qgz_region = 0;  // region size of the last qgZ call
  cudaIpcMemHandle_t handle;
  int device = 0;
  // qgZ stage pipelining: K1 of stage s+1 runs on `side` while K2/K3 of stage
  // s run on the caller's stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_k1 = nullptr, ev_bar = nullptr;
  // qwZ cross-layer prefetch (zpp_qwz_allgather_next): K0 of the next shard,
  // issued on `side` after barrier ev_qbar, completion ev_pf
  cudaEvent_t ev_pf = nullptr, ev_qbar = nullptr;
  bool pf_valid = false;
  const void* pf_ptr = nullptr;
  int64_t pf_len = 0, pf_block = 0;
  int pf_dtype = 0, pf_bits = 0;
  size_t pf_off = 0;
  // stage tracer (zpp_comm_trace): timing events between the launches of the
  // last traced collective, on its stream
  bool trace = false;
  int tr_n = 0;
  int tr_id[kTraceMax] = {};
  cudaEvent_t tr_ev[kTraceMax] = {};

  uint32_t* flag_slot(int owner, int scope, int writer) {
    return reinterpret_cast<uint32_t*>(peers[owner] + sym_bytes) + scope * kMaxRanks + writer;
  }
  // members of a barrier scope, ascending
  std::vector<int> members(int scope) const {
    std::vector<int> m;
    const int node = rank / group, loc = rank % group;
    if (scope == 0) {
      for (int r = 0; r < world; ++r) m.push_back(r);
    } else if (scope == 1) {
      for (int j = 0; j < group; ++j) m.push_back(node * group + j);
    } else {
      for (int c = 0; c < world / group; ++c) m.push_back(c * group + loc);
    }
    return m;
  }
};

static int comm_ok(zpp_comm_t c) {
  if (!c) return fail(ZPP_ERR_VALIDATION, "null communicator");
  for (int r = 0; r < c->world; ++r)
    if (!c->peers[r]) return fail(ZPP_ERR_COMM, "peers not opened (call zpp_comm_open_peers)");
  return ZPP_OK;
}

static int barrier(zpp_comm_t c, int scope, int timeout_ms, uint32_t* flag, cudaStream_t st) {
  std::vector<int> m = c->members(scope);
  if (m.size() == 1) return ZPP_OK;  // nothing to wait for
  const uint32_t e = ++c->epoch[scope];
  BarrierArgs a;
  for (size_t i = 0; i < m.size(); ++i) {
    a.remote[i] = c->flag_slot(m[i], scope, c->rank);
    a.local[i] = c->flag_slot(c->rank, scope, m[i]);
  }
  const uint64_t to = (uint64_t)(timeout_ms > 0 ? timeout_ms : 60000) * 1000000ull;
  launch_k(barrier_kernel, 1, 64, 0, st, a, (int)m.size(), e, to, flag);
  return check_cuda(cudaGetLastError(), "barrier_kernel launch");
}

// stage ids for the tracer: what just finished when the event was recorded
enum TraceId { TR_BEGIN = 0, TR_QUANT = 1, TR_BARRIER = 2, TR_GATHER = 3, TR_K1 = 4, TR_K2 = 5, TR_K3 = 6 };
static void trace_reset(zpp_comm_t c) { c->tr_n = 0; }
static void trace_mark(zpp_comm_t c, int id, cudaStream_t st) {
  if (!c->trace || c->tr_n >= kTraceMax) return;
  if (!c->tr_ev[c->tr_n]) cudaEventCreate(&c->tr_ev[c->tr_n]);
  c->tr_id[c->tr_n] = id;
  cudaEventRecord(c->tr_ev[c->tr_n++], st);
}

static size_t absmax_elem(int dtype) { return dtype == ZPP_F64 ? 8 : 4; }
static const int kBarrierTimeoutMs = 60000;

extern "C" {

int zpp_comm_create(int rank, int world, int group_size, size_t sym_bytes, zpp_comm_t* out) {
  if (!out) return fail(ZPP_ERR_VALIDATION, "null output");
  if (world < 1 || world > kMaxRanks) return fail(ZPP_ERR_VALIDATION, "world must be in [1, 64]");
  if (rank < 0 || rank >= world) return fail(ZPP_ERR_VALIDATION, "rank out of range");
  if (group_size < 1 || world % group_size) return fail(ZPP_ERR_VALIDATION, "group_size must divide world");
  zpp_comm* c = new zpp_comm();
  c->rank = rank;
  c->world = world;
  c->group = group_size;
  c->sym_bytes = align256(sym_bytes);
  cudaGetDevice(&c->device);
  int rc = check_cuda(cudaMalloc(&c->local, c->sym_bytes + kFlagBytes), "cudaMalloc symmetric buffer");
  if (rc) {
    delete c;
    return rc;
  }
  rc = check_cuda(cudaMemset(c->local + c->sym_bytes, 0, kFlagBytes), "flag memset");
  if (!rc) rc = check_cuda(cudaIpcGetMemHandle(&c->handle, c->local), "cudaIpcGetMemHandle");
  if (rc) {
    cudaFree(c->local);
    delete c;
    return rc;
  }
  c->peers[rank] = c->local;
  *out = c;
  return ZPP_OK;
}

int zpp_comm_ipc_handle(zpp_comm_t c, void* handle_out) {
  if (!c || !handle_out) return fail(ZPP_ERR_VALIDATION, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == ZPP_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &c->handle, sizeof(c->handle));
  return ZPP_OK;
}

int zpp_comm_open_peers(zpp_comm_t c, const void* all_handles) {
  if (!c || !all_handles) return fail(ZPP_ERR_VALIDATION, "null argument");
  const uint8_t* h = reinterpret_cast<const uint8_t*>(all_handles);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->peers[r]) continue;
    cudaIpcMemHandle_t hh;
    std::memcpy(&hh, h + (size_t)r * ZPP_IPC_HANDLE_BYTES, sizeof(hh));
    void* p = nullptr;
    int rc = check_cuda(cudaIpcOpenMemHandle(&p, hh, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    if (rc) return rc;
    c->peers[r] = reinterpret_cast<uint8_t*>(p);
    c->opened[r] = true;
  }
  return ZPP_OK;
}

void* zpp_comm_sym_ptr(zpp_comm_t c, int rank) {
  if (!c || rank < 0 || rank >= c->world) return nullptr;
  return c->peers[rank];
}

size_t zpp_comm_sym_bytes(zpp_comm_t c) { return c ? c->sym_bytes : 0; }

int zpp_comm_barrier(zpp_comm_t c, int scope, int timeout_ms, void* errflag, void* stream) {
  int rc = comm_ok(c);
  if (rc) return rc;
  if (scope < 0 || scope >= kScopes) return fail(ZPP_ERR_VALIDATION, "scope must be 0, 1 or 2");
  return barrier(c, scope, timeout_ms, reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream));
}

int zpp_comm_reset(zpp_comm_t c) {
  if (!c) return fail(ZPP_ERR_VALIDATION, "null communicator");
  // The caller has synchronised every rank's device and passed a host barrier
  // (Communicator.recover), so no barrier kernel or peer read is in flight:
  // zero this rank's flag words and restart every epoch and double-buffer
  // phase from the state zpp_comm_create leaves.
  int rc = check_cuda(cudaDeviceSynchronize(), "reset sync");
  if (!rc) rc = check_cuda(cudaMemset(c->local + c->sym_bytes, 0, kFlagBytes), "flag memset");
  if (rc) return rc;
  for (int s = 0; s < kScopes; ++s) c->epoch[s] = 0;
  c->qwz_uses = c->qgz_uses = 0;
  c->qwz_region = c->qgz_region = 0;
  c->pf_valid = false;
  return check_cuda(cudaDeviceSynchronize(), "reset sync");
}

int zpp_comm_destroy(zpp_comm_t c) {
  if (!c) return ZPP_OK;
  cudaDeviceSynchronize();
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_k1) cudaEventDestroy(c->ev_k1);
  if (c->ev_bar) cudaEventDestroy(c->ev_bar);
  if (c->ev_pf) cudaEventDestroy(c->ev_pf);
  if (c->ev_qbar) cudaEventDestroy(c->ev_qbar);
  if (c->side) cudaStreamDestroy(c->side);
  for (int i = 0; i < kTraceMax; ++i)
    if (c->tr_ev[i]) cudaEventDestroy(c->tr_ev[i]);
  for (int r = 0; r < c->world; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->peers[r]);
  cudaFree(c->local);
  delete c;
  return ZPP_OK;
}

// ---------------------------------------------------------------------------
// qwZ

static size_t qwz_region(int64_t shard_len, int bits, int64_t block, int dtype) {
  const int64_t nb = ceil_div(shard_len, block);
  return align256((size_t)code_bytes(shard_len, bits, block)) + align256((size_t)nb * absmax_elem(dtype));
}

size_t zpp_qwz_sym_bytes(int64_t shard_len, int bits, int64_t block, int world) {
  (void)world;
  return 2 * qwz_region(shard_len, bits, block, ZPP_F64);
}

int zpp_qwz_allgather(zpp_comm_t c, size_t sym_offset, const void* shard, int dtype, int64_t shard_len, int bits,
                      int64_t block, void* out, int out_dtype, int64_t out_stride, void* sec_out, int64_t sec_lo,
                      int64_t sec_len, void* errflag, void* stream) {
  return zpp_qwz_allgather_next(c, sym_offset, shard, dtype, shard_len, bits, block, out, out_dtype, out_stride,
                                sec_out, sec_lo, sec_len, nullptr, 0, errflag, stream);
}

// Cross-layer prefetch-quantize ("the communication of the
// current layer and the quantization of the next layer can be launched at the
// same time on different CUDA streams").  With next_shard, K0 of the next
// call's shard runs on the side stream into the next call's half, beside this
// call's NVLink gather (which then leaves kPrefetchSms SMs free for it).
// Safety: K0(i+1) rewrites the half of call i-1, whose readers (every rank's
// gather(i-1)) finished before they reached barrier(i); K0(i+1) is ordered
// after this rank passed barrier(i).  The next call finds the prefetched
// shard by (pointer, length, config, offset) and waits for it instead of
// quantizing; any other shard waits for it and is quantized as usual.
// SM budget of the prefetched K0 in split placement: it must finish under
// the gather it hides behind without starving it.  K0 moves ~3 HBM bytes per
// element at ~6.3 TB/s on the whole GPU; the gather pulls (W-1) code bytes
// per element at ~640 GB/s, so K0 needs about 0.3/(W-1) of the SMs.  Swept
// at W = 2 (profiles/r2/qwz_prefetch_sweep_n2_r2.jsonl): 20 SMs 19.5 ms,
// 40 SMs 14.2, 59 SMs 15.7, 74 SMs 18.2 (no prefetch 14.6): 0.27 of the SMs.
static int qwz_sms_for_prefetch(int world) {
  static const int v = [] {
    const char* e = getenv("ZPP_QWZ_PREFETCH_SMS");
    return e ? atoi(e) : 0;
  }();
  if (v > 0) return v;
  const int s = (int)(sm_count() * 0.27 / std::max(1, world - 1) + 0.5);
  return std::min(std::max(8, s), sm_count() / 2);
}

int zpp_qwz_allgather_next(zpp_comm_t c, size_t sym_offset, const void* shard, int dtype, int64_t shard_len,
                           int bits, int64_t block, void* out, int out_dtype, int64_t out_stride, void* sec_out,
                           int64_t sec_lo, int64_t sec_len, const void* next_shard, int64_t next_len, void* errflag,
                           void* stream) {
  int rc = comm_ok(c);
  if (rc) return rc;
  if ((bits != 4 && bits != 8) || block < 8 || block % 8) return fail(ZPP_ERR_CONFIG, "bad quant config");
  if (shard_len < 0 || (shard_len > 0 && (!shard || !out))) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  if (dtype < 0 || dtype > ZPP_F64 || out_dtype < 0 || out_dtype > ZPP_F64)
    return fail(ZPP_ERR_VALIDATION, "unknown dtype");
  if (next_shard && next_len <= 0) return fail(ZPP_ERR_VALIDATION, "next_len must be positive");
  const size_t region = qwz_region(shard_len, bits, block, ZPP_F64);
  if (sym_offset + 2 * region > c->sym_bytes) return fail(ZPP_ERR_VALIDATION, "symmetric buffer too small for qwZ");
  if (shard_len == 0) return ZPP_OK;
  PdlScope pdl(true);  // K0 -> barrier -> gather overlap their launches
  trace_reset(c);
  trace_mark(c, TR_BEGIN, reinterpret_cast<cudaStream_t>(stream));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* flag = reinterpret_cast<uint32_t*>(errflag);
  // a prefetch issued by the previous call for exactly this shard?
  const bool had_pf = c->pf_valid;
  const bool use_pf = had_pf && c->pf_ptr == shard && c->pf_len == shard_len && c->pf_dtype == dtype &&
                      c->pf_bits == bits && c->pf_block == block && c->pf_off == sym_offset;
  c->pf_valid = false;
  if (had_pf && (rc = check_cuda(cudaStreamWaitEvent(st, c->ev_pf, 0), "wait prefetch"))) return rc;
  // A different shard length moves the half boundaries, so K0 of this call
  // could overwrite codes peers are still pulling for the previous call (a
  // rank passing that call's barrier only proves peers finished its K0, not
  // its gather).  Drain every rank's reads of the old layout first -- the same
  // guard qgZ takes below.
  if (c->world > 1 && c->qwz_region != 0 && c->qwz_region != region) {
    if ((rc = barrier(c, 0, kBarrierTimeoutMs, flag, st))) return rc;
  }
  c->qwz_region = region;
  const uint64_t use = c->qwz_uses++;
  const size_t base = sym_offset + (use & 1) * region;
  const size_t abs_off = align256((size_t)code_bytes(shard_len, bits, block));
  if (c->world == 1 && sec_out == nullptr && out_dtype == dtype) {
    // 1-GPU world: the gather is the local round trip -- one fused pass
    bool handled = false;
    rc = launch_quantize_deq(shard, dtype, shard_len, bits, block, c->local + base, c->local + base + abs_off, out,
                             flag, st, &handled);
    if (rc || handled) return rc;
  }
  if (!use_pf) {
    AddrSpec a;
    a.n = shard_len;
    rc = launch_quantize(shard, dtype, a, shard_len, bits, block, c->local + base, c->local + base + abs_off, flag, st);
    if (rc) return rc;
  }
  trace_mark(c, TR_QUANT, st);
  rc = barrier(c, 0, kBarrierTimeoutMs, flag, st);
  if (rc) return rc;
  trace_mark(c, TR_BARRIER, st);
  // prefetch: K0 of the next shard into the next call's half, on the side
  // stream, after this rank passed barrier(i); only for an unchanged layout.
  // Two placements (40-layer GPT-13B forward, profiles/r2/qwz_prefetch_sweep*):
  //  * share (W >= 3): both grids span every SM, the gather capped at
  //    ZPP_QWZ_GATHER_OCC = 3 CTAs per SM (of 4) and K0 at one CTA per SM, so
  //    K0 runs in the issue slots the NVLink-bound gather leaves idle.  W = 4:
  //    16.1 ms vs 17.6 ms without prefetch (occupancy 2: 18.4; 1: 30.3;
  //    split with 20 SMs: 16.3);
  //  * split (W = 2): K0 on its own ZPP_QWZ_PREFETCH_SMS = 40 SMs, the gather
  //    on the rest: 14.2 ms vs 14.6 ms (share at occupancy 2: 18.2 -- the
  //    W = 2 gather needs its full occupancy).
  // ZPP_QWZ_PREFETCH_MODE=share|split overrides.
  static const int pf_mode_env = [] {
    const char* e = getenv("ZPP_QWZ_PREFETCH_MODE");
    return !e ? 0 : (e[0] == 's' && e[1] == 'p') ? 2 : 1;  // 1 share, 2 split
  }();
  const bool pf_split = pf_mode_env == 2 || (pf_mode_env == 0 && c->world == 2);
  static const int gather_occ = [] {
    const char* e = getenv("ZPP_QWZ_GATHER_OCC");
    return e ? atoi(e) : 3;
  }();
  const bool prefetch = next_shard && c->world > 1 && qwz_region(next_len, bits, block, ZPP_F64) == region;
  if (prefetch) {
    if (!c->side && (rc = check_cuda(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream")))
      return rc;
    if (!c->ev_pf && (rc = check_cuda(cudaEventCreateWithFlags(&c->ev_pf, cudaEventDisableTiming), "event")))
      return rc;
    if (!c->ev_qbar && (rc = check_cuda(cudaEventCreateWithFlags(&c->ev_qbar, cudaEventDisableTiming), "event")))
      return rc;
    if ((rc = check_cuda(cudaEventRecord(c->ev_qbar, st), "record"))) return rc;
  }
  const void* codes[kMaxRanks];
  const void* absmax[kMaxRanks];
  for (int r = 0; r < c->world; ++r) {
    codes[r] = c->peers[r] + base;
    absmax[r] = c->peers[r] + base + abs_off;
  }
  {  // the gather is enqueued first, so its CTAs are placed first
    SmBudget budget(prefetch && pf_split ? sm_count() - qwz_sms_for_prefetch(c->world) : 0);
    OccCap cap(prefetch && !pf_split ? gather_occ : 0);
    rc = launch_gather_dequant(codes, absmax, dtype == ZPP_F64 ? ZPP_F64 : ZPP_F32, c->world, c->rank, shard_len,
                               bits, block, out, out_dtype, sec_out, sec_lo, sec_len, flag, st, out_stride);
  }
  if (rc) return rc;
  if (prefetch) {
    if ((rc = check_cuda(cudaStreamWaitEvent(c->side, c->ev_qbar, 0), "wait"))) return rc;
    const size_t nbase = sym_offset + ((use + 1) & 1) * region;
    const size_t nabs = align256((size_t)code_bytes(next_len, bits, block));
    AddrSpec a;
    a.n = next_len;
    {
      SmBudget budget(pf_split ? qwz_sms_for_prefetch(c->world) : 0);
      OccCap cap(pf_split ? 0 : 1);
      rc = launch_quantize(next_shard, dtype, a, next_len, bits, block, c->local + nbase, c->local + nbase + nabs, flag,
                           c->side);
    }
    if (rc) return rc;
    if ((rc = check_cuda(cudaEventRecord(c->ev_pf, c->side), "record"))) return rc;
    c->pf_valid = true;
    c->pf_ptr = next_shard;
    c->pf_len = next_len;
    c->pf_dtype = dtype;
    c->pf_bits = bits;
    c->pf_block = block;
    c->pf_off = sym_offset;
  }
  trace_mark(c, TR_GATHER, st);
  return rc;
}

// ---------------------------------------------------------------------------
// hpZ

size_t zpp_hpz_sym_bytes(int64_t sec_len, int elem_bytes) { return align256((size_t)sec_len * elem_bytes); }

int zpp_hpz_allgather(zpp_comm_t c, size_t sym_offset, int64_t sec_len, int elem_bytes, void* out, void* errflag,
                      void* stream) {
  int rc = comm_ok(c);
  if (rc) return rc;
  if (sec_len < 0 || elem_bytes <= 0 || (sec_len > 0 && !out)) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  const int64_t seg = sec_len * elem_bytes;
  if (sym_offset + (size_t)seg > c->sym_bytes) return fail(ZPP_ERR_VALIDATION, "symmetric buffer too small for hpZ");
  if (seg == 0) return ZPP_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PdlScope pdl(true);  // barrier -> gather overlap their launches
  rc = barrier(c, 1, kBarrierTimeoutMs, reinterpret_cast<uint32_t*>(errflag), st);
  if (rc) return rc;
  std::vector<int> m = c->members(1);
  SrcTable t;
  std::memset(&t, 0, sizeof(t));
  for (size_t i = 0; i < m.size(); ++i) t.codes[i] = c->peers[m[i]] + sym_offset;
  const int vec = (seg % 16 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && (sym_offset % 16 == 0);
  const int n = (int)m.size();
  if (vec) {
    const int smem = kCopyStages * kCopyTile + kCopyStages * 8;
    cudaFuncSetAttribute(gather_copy_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_copy_tma_kernel, 256, smem);
    const int64_t tiles = ceil_div(seg, kCopyTile) * n;
    const int grid = (int)std::min<int64_t>((int64_t)sm_count() * std::max(occ, 1), tiles);
    launch_k(gather_copy_tma_kernel, grid, 256, smem, st, t, n, c->rank % c->group, seg, reinterpret_cast<uint8_t*>(out),
                                                    reinterpret_cast<const uint32_t*>(errflag));
    return check_cuda(cudaGetLastError(), "gather_copy_tma_kernel launch");
  }
  const int grid = (int)std::min<int64_t>(4 * sm_count(), std::max<int64_t>(1, ceil_div(seg * n, 16 * 256)));
  launch_k(gather_copy_kernel, grid, 256, 0, st, t, n, c->rank % c->group, seg, reinterpret_cast<uint8_t*>(out), vec,
                                           reinterpret_cast<const uint32_t*>(errflag));
  return check_cuda(cudaGetLastError(), "gather_copy_kernel launch");
}

// ---------------------------------------------------------------------------
// qgZ

struct QgzLayout {
  int64_t L;
  size_t send_codes, send_abs, hop_codes, hop_abs, ws, region;
};

static QgzLayout qgz_layout(int64_t n, int world, int Y, int stages, int ib, int64_t iblk, int ob, int64_t oblk) {
  QgzLayout l;
  l.L = n / ((int64_t)stages * world);
  const int64_t send_elems = (int64_t)world * l.L;
  const int64_t hop_elems = (int64_t)Y * l.L;
  size_t off = 0;
  l.send_codes = off;
  off += align256((size_t)code_bytes(send_elems, ib, iblk));
  l.send_abs = off;
  off += align256((size_t)ceil_div(send_elems, iblk) * 8);
  l.hop_codes = off;
  off += align256((size_t)code_bytes(hop_elems, ob, oblk));
  l.hop_abs = off;
  off += align256((size_t)ceil_div(hop_elems, oblk) * 8);
  l.ws = off;
  off += align256(drq_has_reg_path(oblk) ? 0 : drq_workspace_bytes(hop_elems, oblk));
  l.region = off;
  return l;
}

size_t zpp_qgz_sym_bytes(int64_t n, int world, int stages, int intra_bits, int64_t intra_block, int inter_bits,
                         int64_t inter_block) {
  if (world < 1 || stages < 1 || intra_block < 8 || inter_block < 8) return 0;
  return 2 * qgz_layout(n, world, world, stages, intra_bits, intra_block, inter_bits, inter_block).region;
}

int zpp_qgz_reduce_scatter(zpp_comm_t c, size_t sym_offset, const void* grad, int dtype, int64_t n, int stages,
                           int reorder, int intra_bits, int64_t intra_block, int inter_bits, int64_t inter_block,
                           void* out, int out_dtype, void* errflag, void* stream) {
  return zpp_qgz_reduce_scatter_buckets(c, sym_offset, grad, dtype, n, 1, stages, reorder, intra_bits, intra_block,
                                        inter_bits, inter_block, out, out_dtype, errflag, stream);
}

int zpp_qgz_reduce_scatter_buckets(zpp_comm_t c, size_t sym_offset, const void* grad, int dtype, int64_t n,
                                   int n_buckets, int stages, int reorder, int intra_bits, int64_t intra_block,
                                   int inter_bits, int64_t inter_block, void* out, int out_dtype, void* errflag,
                                   void* stream) {
  int rc = comm_ok(c);
  if (rc) return rc;
  if ((intra_bits != 4 && intra_bits != 8) || (inter_bits != 4 && inter_bits != 8) || intra_block < 8 ||
      intra_block % 8 || inter_block < 8 || inter_block % 8)
    return fail(ZPP_ERR_CONFIG, "bad quant config");
  if (stages < 1) return fail(ZPP_ERR_VALIDATION, "stages must be >= 1");
  if (n_buckets < 1) return fail(ZPP_ERR_VALIDATION, "n_buckets must be >= 1");
  const int W = c->world, X = c->group, Y = W / X;
  if (n < 0 || n % ((int64_t)stages * W)) return fail(ZPP_ERR_VALIDATION, "input length not divisible by stages*world");
  const QgzLayout l = qgz_layout(n, W, Y, stages, intra_bits, intra_block, inter_bits, inter_block);
  if (l.L % intra_block || l.L % inter_block)
    return fail(ZPP_ERR_VALIDATION, "slice length is not a multiple of block_size");
  if (sym_offset + 2 * l.region > c->sym_bytes) return fail(ZPP_ERR_VALIDATION, "symmetric buffer too small for qgZ");
  if (n == 0) return ZPP_OK;
  if (!grad || !out) return fail(ZPP_ERR_VALIDATION, "null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* flag = reinterpret_cast<uint32_t*>(errflag);
  const int node = c->rank / X, loc = c->rank % X;
  const int in_abs = dtype == ZPP_F64 ? ZPP_F64 : ZPP_F32;
  const size_t in_abs_sz = absmax_elem(in_abs);
  const size_t out_esz = out_dtype == ZPP_F64 ? 8 : (out_dtype == ZPP_F32 ? 4 : 2);
  const int64_t L = l.L;
  const int64_t msg_elems = (int64_t)Y * L;  // one hop-1 message
  const size_t in_esz = dtype == ZPP_F64 ? 8 : (dtype == ZPP_F32 ? 4 : 2);
  // Work units u = (bucket b, stage s), b-major: K1 of unit u+1 runs on the
  // side stream beside K2/K3 of unit u.  Buckets are independent qgz_2hop
  // calls (bucket b: grad[b*n, (b+1)*n) -> out[b*n/W, (b+1)*n/W)); pipelining
  // them needs no extra barrier, unlike stages of one bucket.
  // ZPP_QGZ_XB=0 runs buckets back to back without overlap (A/B).
  static const int xb_env = [] {
    const char* e = getenv("ZPP_QGZ_XB");
    return e ? atoi(e) : 1;
  }();
  const int units = n_buckets * stages;
  // Bucket pipelining pays only when hop 2 is a self-send (Y = 1, pull K2):
  // 8 x 256 MiB buckets (profiles/r2/qgz_bucket_pipeline_sweep_r2.jsonl),
  // 1x4: 145.6 us per bucket vs 171.9 back to back; 1x2: 175.5 vs 182.7.
  // With a second hop (push K1 + K2 + cross barrier + K3) every split lost
  // (2x2: 216-273 vs 210.6), so those buckets run back to back, and so do
  // the buckets of a 1-GPU world (no NVLink wait to hide: 7B stream 15.7 vs
  // 11.6 ms).
  // ZPP_QGZ_XB=0 disables it, ZPP_QGZ_XB=2 forces it (A/B).
  const bool xb = n_buckets > 1 && (xb_env == 2 || (xb_env == 1 && Y == 1 && X > 1));
  const bool pipelined = stages > 1 || xb;
  if (pipelined && !c->ev_start) {
    if (!c->side) rc = check_cuda(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
    if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming), "event");
    if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&c->ev_k1, cudaEventDisableTiming), "event");
    if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&c->ev_bar, cudaEventDisableTiming), "event");
    if (rc) return rc;
  }
  // a different region size (another n or config) moves the half boundaries:
  // drain every rank's reads of the previous layout first
  if (c->qgz_region != 0 && c->qgz_region != l.region) {
    if ((rc = barrier(c, 0, kBarrierTimeoutMs, flag, st))) return rc;
  }
  c->qgz_region = l.region;
  PdlScope pdl(true);  // K1 -> barrier -> K2 -> barrier -> K3 overlap their launches
  trace_reset(c);
  trace_mark(c, TR_BEGIN, st);
  const uint64_t use0 = c->qgz_uses;
  c->qgz_uses += units;
  auto base_of = [&](int u) { return sym_offset + ((use0 + u) & 1) * l.region; };
  // unit u = (bucket u / stages, stage u % stages) writes out[u*L, (u+1)*L):
  // bucket b's partition (n/W = stages*L elements) follows bucket b-1's
  auto out_of = [&](int u) { return reinterpret_cast<uint8_t*>(out) + (size_t)u * L * out_esz; };
  // K1: swizzle + quantize stage s's slices into my send buffer [j][c][e]
  // SM split while K1(s+1) runs beside K2(s) (pipelined only)
  static const int k1_sms_env = [] {
    const char* e = getenv("ZPP_QGZ_K1_SMS");
    return e ? atoi(e) : 0;
  }();
  static const int k1_xb_sms_env = [] {
    const char* e = getenv("ZPP_QGZ_K1_XB_SMS");
    return e ? atoi(e) : 0;
  }();
  // SMs (resident-CTA budget) of the K1 running beside a K2/K3: a third when
  // overlapping stages of one bucket (K2/K3 of a stage are short), a larger
  // share across buckets (K1 and the fold are both issue-bound; swept in
  // tools/qgz_xb_sweep.sh)
  // ZPP_QGZ_XB_MODE=share: across buckets, K1(b+1) and K2/K3(b) both span
  // every SM instead (K1 one CTA per SM, the fold ZPP_QGZ_K2_OCC = 2 CTAs
  // per SM), sharing each SM's issue slots
  static const int xb_share = [] {
    const char* e = getenv("ZPP_QGZ_XB_MODE");
    return e && e[0] == 's' && e[1] == 'h';
  }();
  static const int k2_occ_env = [] {
    const char* e = getenv("ZPP_QGZ_K2_OCC");
    return e ? atoi(e) : 2;
  }();
  const bool share = pipelined && stages == 1 && xb_share;
  const int k1_sms = !pipelined || share ? 0
                     : stages > 1 ? (k1_sms_env > 0 ? k1_sms_env : sm_count() / 3)
                                  : (k1_xb_sms_env > 0 ? k1_xb_sms_env : (X >= 4 ? sm_count() / 2 : sm_count() * 2 / 5));
  // Hop 1 either
  //  * push: K1 (quantize_push_kernel) streams each message into the receiving
  //    peer's [src_loc][c][e] region with TMA bulk stores while it quantizes,
  //    and K2 folds local HBM; or
  //  * pull: K1 writes the local send buffer and K2 (drq_tma_kernel) pulls the
  //    X messages over NVLink while it folds.
  // Measured on 4 B200s (profiles/r2/qgz_push_pull_r2.md), 256 MiB bf16
  // bucket: 2x2 push 237 us vs pull 246 us; 1x4 push 195 us vs pull 187 us
  // (with one group K2 also writes the fp32 partition, and its NVLink pull
  // hides under that work), so push is used when there is a second hop
  // (Y > 1) and K1 has a register path.  ZPP_QGZ_MODE=push|pull overrides
  // (development A/B).  The choice depends only on arguments every rank shares.
  const size_t msg_code_bytes = (size_t)code_bytes(msg_elems, intra_bits, intra_block);
  const int64_t msg_blocks = msg_elems / intra_block;
  static const int mode_env = [] {
    const char* e = getenv("ZPP_QGZ_MODE");
    if (!e) e = getenv("ZPP_QGZ_PULL") && getenv("ZPP_QGZ_PULL")[0] == '1' ? "pull" : nullptr;
    return !e ? 0 : (e[1] == 'u' && e[2] == 's') ? 1 : 2;  // 1 push, 2 pull
  }();
  const int64_t epl = dtype == ZPP_F32 ? 32 : 64;
  const bool want_push = mode_env == 1 || (mode_env == 0 && Y > 1);
  // Hop 2 by push (K2 stores into the receivers' slots, K3 local) is opt-in
  // (ZPP_QGZ_HOP2=push): measured no faster at 2x2 (193.2 vs 193.5 us per
  // 256 MiB bucket) and slower at 2x1 (270 vs 255 us) than K3 pulling the
  // segment with TMA (profiles/r2/qgz_hop2_push_r2.jsonl).
  static const int hop2_env = [] {
    const char* e = getenv("ZPP_QGZ_HOP2");
    return !e ? 0 : (e[1] == 'u' && e[2] == 's') ? 1 : 2;  // 1 push, 2 pull
  }();
  const bool hop2_push = hop2_env == 1;
  const bool push = want_push && dtype != ZPP_F64 && X <= 8 && intra_block % epl == 0 &&
                    intra_block / epl >= 2 && intra_block / epl <= 32 &&
                    ((intra_block / epl) & (intra_block / epl - 1)) == 0;
  if (push && (reinterpret_cast<uintptr_t>(grad) & 15))
    return fail(ZPP_ERR_VALIDATION, "qgZ: the gradient buffer must be 16-byte aligned");
  auto k1 = [&](int u, cudaStream_t on) {
    SmBudget budget(u > 0 ? k1_sms : 0);  // K1(0) runs alone
    OccCap cap(u > 0 && share ? 1 : 0);
    const int s = u % stages;
    const void* g = reinterpret_cast<const uint8_t*>(grad) + (size_t)(u / stages) * n * in_esz;
    AddrSpec a;
    a.swizzle = true;
    a.L = L;
    a.part = (int64_t)stages * L;
    a.stage_off = (int64_t)s * L;
    a.X = X;
    a.Y = Y;
    a.reorder = reorder ? 1 : 0;
    const size_t base = base_of(u);
    if (push) {
      uint8_t* dc[kMaxPush];
      uint8_t* da[kMaxPush];
      for (int j = 0; j < X; ++j) {
        uint8_t* p = c->peers[node * X + j] + base;
        dc[j] = p + l.send_codes + msg_code_bytes * loc;
        da[j] = p + l.send_abs + (size_t)msg_blocks * in_abs_sz * loc;
      }
      bool handled = false;
      // rank loc starts with the message for local peer loc+1: the group's
      // ranks begin on different destinations
      const int rc1 = launch_quantize_push(g, dtype, a, (int64_t)W * L, intra_bits, intra_block, dc, da, msg_blocks,
                                           (loc + 1) % X, loc, flag, on, &handled);
      if (rc1 || handled) return rc1;
      return fail(ZPP_ERR_VALIDATION, "qgZ: no push path for this shape");
    }
    return launch_quantize(g, dtype, a, (int64_t)W * L, intra_bits, intra_block, c->local + base + l.send_codes,
                           c->local + base + l.send_abs, flag, on);
  };
  if (pipelined) {
    // K1(s) rewrites the send half used by stage s-2, whose readers (group
    // peers' K2(s-2)) all finished before they reached group barrier(s-1);
    // so K1(s) only waits for that barrier, and overlaps K2/K3(s-1).
    if ((rc = check_cuda(cudaEventRecord(c->ev_start, st), "record"))) return rc;
    if ((rc = check_cuda(cudaStreamWaitEvent(c->side, c->ev_start, 0), "wait"))) return rc;
    if ((rc = k1(0, c->side))) return rc;
    if ((rc = check_cuda(cudaEventRecord(c->ev_k1, c->side), "record"))) return rc;
  }
  for (int s = 0; s < units; ++s) {
    const size_t base = base_of(s);
    uint8_t* const out_s = out_of(s);
    if (pipelined) {
      if ((rc = check_cuda(cudaStreamWaitEvent(st, c->ev_k1, 0), "wait"))) return rc;
    } else if ((rc = k1(s, st))) {
      return rc;
    }
    trace_mark(c, TR_K1, st);
    rc = barrier(c, 1, kBarrierTimeoutMs, flag, st);
    if (rc) return rc;
    trace_mark(c, TR_BARRIER, st);
    if (pipelined && s + 1 < units) {
      if ((rc = check_cuda(cudaEventRecord(c->ev_bar, st), "record"))) return rc;
      if ((rc = check_cuda(cudaStreamWaitEvent(c->side, c->ev_bar, 0), "wait"))) return rc;
      if ((rc = k1(s + 1, c->side))) return rc;
      if ((rc = check_cuda(cudaEventRecord(c->ev_k1, c->side), "record"))) return rc;
    }
    SmBudget budget(pipelined && !share && s + 1 < units ? sm_count() - k1_sms : 0);
    OccCap cap(share && s + 1 < units ? k2_occ_env : 0);
    // K2: the X messages for this rank, ascending local source -- pushed into
    // this rank's receive region by the group's K1s, or pulled from the peers
    const void* codes[kMaxRanks];
    const void* absmax[kMaxRanks];
    for (int j = 0; j < X; ++j) {
      if (push) {
        const uint8_t* p = c->local + base;
        codes[j] = p + l.send_codes + msg_code_bytes * j;
        absmax[j] = p + l.send_abs + (size_t)msg_blocks * in_abs_sz * j;
      } else {
        const uint8_t* p = c->peers[node * X + j] + base;
        codes[j] = p + l.send_codes + msg_code_bytes * loc;
        absmax[j] = p + l.send_abs + (size_t)msg_blocks * in_abs_sz * loc;
      }
    }
    if (Y == 1) {  // hop 2 is a self-send: K2 writes the final partition directly
      bool handled = false;
      if (in_abs == ZPP_F32 && !push)
        rc = launch_drq_tma(codes, absmax, X, msg_elems, intra_bits, intra_block, inter_bits, inter_block, nullptr,
                            reinterpret_cast<double*>(c->local + base + l.hop_abs),
                            out_s, out_dtype, flag, st, &handled);
      if (rc) return rc;
      if (handled) {
        trace_mark(c, TR_K2, st);
        continue;
      }
      rc = launch_drq_final(codes, absmax, in_abs, X, msg_elems, intra_bits, intra_block, inter_bits, inter_block,
                            reinterpret_cast<double*>(c->local + base + l.hop_abs),
                            out_s, out_dtype, flag, st, &handled);
      if (rc) return rc;
      if (handled) {
        trace_mark(c, TR_K2, st);
        continue;
      }
    }
    bool handled = false;
    // One GPU per group with one codec for both hops: hop 2 sends K1's codes
    // as they are (hop_absmax_x1_kernel has the proof) and only the f64
    // absmax is computed; ZPP_QGZ_X1=0 runs the full K2 (A/B)
    static const int x1_env = [] {
      const char* e = getenv("ZPP_QGZ_X1");
      return e ? atoi(e) : 1;
    }();
    // Not when pipelined: K3 of the cross peers then reads this rank's send
    // region, whose half K1(s+1) would rewrite right after the (single-member,
    // skipped) group barrier(s), before the peers' K3(s-1) is known done.
    const bool x1 = x1_env != 0 && !pipelined && X == 1 && intra_bits == inter_bits &&
                    intra_block == inter_block && in_abs == ZPP_F32;
    if (x1) {
      const int64_t nb = msg_elems / inter_block;
      const float* m32 = reinterpret_cast<const float*>(c->local + base + l.send_abs);
      double* m64 = reinterpret_cast<double*>(c->local + base + l.hop_abs);
      const int grid = (int)std::min<int64_t>(4 * sm_count(), std::max<int64_t>(1, ceil_div(nb, 256)));
      if (inter_bits == 4) launch_k(hop_absmax_x1_kernel<7>, grid, 256, 0, st, m32, nb, m64, flag);
      else launch_k(hop_absmax_x1_kernel<127>, grid, 256, 0, st, m32, nb, m64, flag);
      if ((rc = check_cuda(cudaGetLastError(), "hop_absmax_x1_kernel launch"))) return rc;
      handled = true;
    }
    // Hop 2 by push (with a pushed hop 1): K2 stores segment c of its output
    // straight into rank (c, loc)'s hop-2 receive slot for this node, over
    // NVLink, and K3 folds local HBM.  The slot was last read by that rank's
    // K3 of the unit before the previous one, which precedes its cross
    // barrier of the previous unit, which this K2 follows.
    bool hop2_pushed = false;
    if (!x1 && push && hop2_push) {
      HopDst hd{};
      const size_t seg_code_bytes = (size_t)code_bytes(L, inter_bits, inter_block);
      for (int g = 0; g < Y; ++g) {
        uint8_t* p = c->peers[g * X + loc] + base;
        hd.codes[g] = p + l.hop_codes + seg_code_bytes * node;
        hd.absmax[g] = reinterpret_cast<double*>(p + l.hop_abs + (size_t)(L / inter_block) * 8 * node);
      }
      hd.seg_blocks = L / 512;
      rc = launch_drq_hop(codes, absmax, X, msg_elems, intra_bits, intra_block, inter_bits, inter_block, hd, flag, st,
                          &hop2_pushed);
      if (rc) return rc;
      handled = hop2_pushed;
    }
    if (!handled && in_abs == ZPP_F32 && !push)
      rc = launch_drq_tma(codes, absmax, X, msg_elems, intra_bits, intra_block, inter_bits, inter_block,
                          c->local + base + l.hop_codes, reinterpret_cast<double*>(c->local + base + l.hop_abs),
                          nullptr, 0, flag, st, &handled);
    if (rc) return rc;
    if (!handled)
      rc = launch_drq(codes, absmax, in_abs, X, msg_elems, intra_bits, intra_block, inter_bits, inter_block,
                      c->local + base + l.hop_codes, reinterpret_cast<double*>(c->local + base + l.hop_abs),
                      c->local + base + l.ws, drq_workspace_bytes(msg_elems, inter_block), flag, st,
                      /*validate=*/false);
    if (rc) return rc;
    trace_mark(c, TR_K2, st);
    rc = barrier(c, 2, kBarrierTimeoutMs, flag, st);
    if (rc) return rc;
    trace_mark(c, TR_BARRIER, st);
    // K3: segment `node` from the rank with my local index in every group --
    // already in my hop-2 slots [g] when hop 2 was pushed, else pulled
    for (int g = 0; g < Y; ++g) {
      const uint8_t* p = hop2_pushed ? c->local + base : c->peers[g * X + loc] + base;
      const int slot = hop2_pushed ? g : node;
      // X = 1: the segment's codes are K1's, in the send region ([0][c][e])
      codes[g] = p + (x1 ? l.send_codes : l.hop_codes) + (size_t)code_bytes(L, inter_bits, inter_block) * slot;
      absmax[g] = p + l.hop_abs + (size_t)(L / inter_block) * 8 * slot;
    }
    handled = false;
    if (!hop2_pushed)
      rc = launch_dr_tma(codes, absmax, Y, L, inter_bits, inter_block, out_s, out_dtype, flag, st, &handled);
    if (rc) return rc;
    if (!handled)
      rc = launch_dequant_reduce(codes, absmax, ZPP_F64, Y, L, inter_bits, inter_block,
                                 out_s, out_dtype, 1.0, flag,
                                 st, /*validate=*/false);
    if (rc) return rc;
    trace_mark(c, TR_K3, st);
  }
  return ZPP_OK;
}

int zpp_comm_trace(zpp_comm_t c, int enable) {
  if (!c) return fail(ZPP_ERR_VALIDATION, "null communicator");
  c->trace = enable != 0;
  c->tr_n = 0;
  return ZPP_OK;
}

int zpp_comm_trace_read(zpp_comm_t c, int* ids, float* ms, int max) {
  if (!c || (max > 0 && (!ids || !ms))) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  const int n = c->tr_n < max ? c->tr_n : max;
  if (n == 0) return 0;
  int rc = check_cuda(cudaEventSynchronize(c->tr_ev[n - 1]), "trace sync");
  if (rc) return -rc;
  for (int i = 0; i < n; ++i) {
    ids[i] = c->tr_id[i];
    ms[i] = 0.0f;
    if (i > 0 && (rc = check_cuda(cudaEventElapsedTime(&ms[i], c->tr_ev[0], c->tr_ev[i]), "trace elapsed")))
      return -rc;
  }
  return n;
}

}  // extern "C"
