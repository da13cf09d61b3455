// NVLink peer bandwidth probe (one process, all visible GPUs, peer access):
// every GPU moves S bytes to/from each of the other GPUs at once, by
//   pull:      16-byte ld.global from peers' buffers, st to local
//   push:      16-byte ld.global local, st.global to peers' buffers
//   pull_tma:  cp.async.bulk peer -> shared ring -> local stores
// and reports per-GPU ingress GB/s (bytes received / time, max over GPUs).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/p2p_bw tools/p2p_bw.cu && /tmp/p2p_bw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(err_)); return 1; } } while (0)

struct Ptrs { const uint4* src[8]; uint4* dst[8]; };

__global__ void copy_kernel(Ptrs p, int n, size_t units) {
  // n segments; segment s: dst[s][i] = src[s][i]
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int s = 0; s < n; ++s)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < units; i += stride) {
      uint4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = (i + k * stride < units) ? p.src[s][i + k * stride] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) if (i + k * stride < units) p.dst[s][i + k * stride] = v[k];
      i += 3 * stride;
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes) : "memory");
}

constexpr int ST = 4, TILE = 16384;
__global__ void tma_kernel(Ptrs p, int n, size_t bytes, int store_tma) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[ST];
  const int tid = threadIdx.x;
  const int tiles = (int)(bytes / TILE), total = tiles * n;
  if (tid == 0) { for (int i = 0; i < ST; ++i) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int G = gridDim.x;
  auto issue = [&](int g, int slot) {
    if (g < total) {
      const int s = g % n, t = g / n;
      mbar_expect_tx(&bar[slot], TILE);
      bulk_g2s(sm + slot * TILE, reinterpret_cast<const uint8_t*>(p.src[s]) + (size_t)t * TILE, TILE, &bar[slot]);
    }
  };
  if (tid == 0) for (int k = 0; k < ST - 1; ++k) issue(blockIdx.x + k * G, k);
  int k = 0;
  for (int g = blockIdx.x; g < total; g += G, ++k) {
    const int slot = k % ST;
    if (tid == 0) {
      if (store_tma) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(g + (ST - 1) * G, (k + ST - 1) % ST);
    }
    mbar_wait(&bar[slot], (k / ST) & 1);
    const int s = g % n, t = g / n;
    uint8_t* dst = reinterpret_cast<uint8_t*>(p.dst[s]) + (size_t)t * TILE;
    if (store_tma) {
      if (tid == 0) { bulk_s2g(dst, sm + slot * TILE, TILE); asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(sm + slot * TILE);
      for (int i = tid; i < TILE / 16; i += blockDim.x) reinterpret_cast<uint4*>(dst)[i] = src[i];
    }
    __syncthreads();
  }
  if (store_tma && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const size_t S = 256ull << 20;  // bytes per peer pair
  std::vector<uint8_t*> send(ng), recv(ng);
  std::vector<cudaStream_t> st(ng);
  for (int d = 0; d < ng; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < ng; ++e) if (e != d) CK(cudaDeviceEnablePeerAccess(e, 0));
    CK(cudaMalloc(&send[d], S * ng));
    CK(cudaMalloc(&recv[d], S * ng));
    CK(cudaMemset(send[d], d, S * ng));
    CK(cudaStreamCreate(&st[d]));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * TILE));
  }
  const char* names[] = {"pull (ld peer, st local)", "push (ld local, st peer)", "pull_tma (bulk peer->smem, st local)",
                         "push_tma (bulk local->smem, bulk smem->peer)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int G : {148, 296, 592}) {
      float worst = 0;
      for (int rep = 0; rep < 3; ++rep) {
        std::vector<cudaEvent_t> a(ng), b(ng);
        for (int d = 0; d < ng; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        for (int d = 0; d < ng; ++d) {
          CK(cudaSetDevice(d));
          Ptrs p{};
          int n = 0;
          for (int e = 0; e < ng; ++e) {
            if (e == d) continue;
            if (mode == 0 || mode == 2) {  // d receives from e
              p.src[n] = reinterpret_cast<const uint4*>(send[e] + S * d);
              p.dst[n] = reinterpret_cast<uint4*>(recv[d] + S * e);
            } else {  // d sends to e
              p.src[n] = reinterpret_cast<const uint4*>(send[d] + S * e);
              p.dst[n] = reinterpret_cast<uint4*>(recv[e] + S * d);
            }
            ++n;
          }
          CK(cudaEventCreate(&a[d]));
          CK(cudaEventCreate(&b[d]));
          CK(cudaEventRecord(a[d], st[d]));
          if (mode < 2) copy_kernel<<<G, 256, 0, st[d]>>>(p, n, S / 16);
          else tma_kernel<<<G, 256, ST * TILE, st[d]>>>(p, n, S, mode == 3);
          CK(cudaGetLastError());
          CK(cudaEventRecord(b[d], st[d]));
        }
        float mx = 0;
        for (int d = 0; d < ng; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(b[d]));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a[d], b[d]));
          mx = ms > mx ? ms : mx;
        }
        if (rep > 0) worst = mx > worst ? mx : worst;
      }
      const double gbs = (double)S * (ng - 1) / (worst * 1e-3) / 1e9;
      printf("%d GPUs  %-44s grid %4d: %.3f ms  ingress %.0f GB/s per GPU\n", ng, names[mode], G, worst, gbs);
    }
  }
  // copy engines: one cudaMemcpyAsync per peer on its own stream (pull: the
  // receiving device's streams read the peer; push: the sender's streams write)
  std::vector<std::vector<cudaStream_t>> ps(ng, std::vector<cudaStream_t>(ng));
  for (int d = 0; d < ng; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < ng; ++e) CK(cudaStreamCreateWithFlags(&ps[d][e], cudaStreamNonBlocking));
  }
  for (int push = 0; push < 2; ++push) {
    float worst = 0;
    for (int rep = 0; rep < 4; ++rep) {
      std::vector<cudaEvent_t> a(ng), b(ng);
      for (int d = 0; d < ng; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < ng; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventCreate(&a[d]));
        CK(cudaEventCreate(&b[d]));
        CK(cudaEventRecord(a[d], st[d]));
        for (int e = 0; e < ng; ++e) {
          if (e == d) continue;
          CK(cudaStreamWaitEvent(ps[d][e], a[d], 0));
          if (!push) CK(cudaMemcpyAsync(recv[d] + S * e, send[e] + S * d, S, cudaMemcpyDeviceToDevice, ps[d][e]));
          else CK(cudaMemcpyAsync(recv[e] + S * d, send[d] + S * e, S, cudaMemcpyDeviceToDevice, ps[d][e]));
          cudaEvent_t j;
          CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
          CK(cudaEventRecord(j, ps[d][e]));
          CK(cudaStreamWaitEvent(st[d], j, 0));
        }
        CK(cudaEventRecord(b[d], st[d]));
      }
      float mx = 0;
      for (int d = 0; d < ng; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(b[d]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a[d], b[d]));
        mx = ms > mx ? ms : mx;
      }
      if (rep > 0) worst = mx > worst ? mx : worst;
    }
    const double gbs = (double)S * (ng - 1) / (worst * 1e-3) / 1e9;
    printf("%d GPUs  %-44s          : %.3f ms  ingress %.0f GB/s per GPU\n", ng,
           push ? "push_ce (cudaMemcpyAsync per peer, sender)" : "pull_ce (cudaMemcpyAsync per peer, receiver)", worst,
           gbs);
  }
  return 0;
}
