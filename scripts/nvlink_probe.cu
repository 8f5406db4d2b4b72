// nvlink_probe.cu -- which access pattern saturates NVLink 5 on this B200 box?
// One process, peer access enabled between all visible GPUs.  Every GPU runs the
// same kernel at the same time (launched back to back from this host thread, each on
// its own device, so nothing waits on another kernel); per-GPU time by CUDA events.
//   pull   : each GPU reads its slice from K peers (ld.global.cg / plain / volatile)
//   push   : each GPU writes its slice to K peers (st.global)
//   bulk   : each GPU pulls with cp.async.bulk (TMA) into shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

struct Ptrs { const float4* src[8]; float4* dst[8]; };

template <int UNROLL, int MODE>  // MODE 0 plain, 1 .cg
__global__ void pull_kernel(Ptrs p, int k_peers, int64_t nvec_per_peer, float4* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int k = 0; k < k_peers; ++k) {
    const float4* s = p.src[k];
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < nvec_per_peer; i += UNROLL * stride) {
      float4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (MODE == 1) v[u] = __ldcg(s + i + u * stride);
        else v[u] = s[i + u * stride];
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  if (acc.x == 12345.f) out[0] = acc;
}

template <int UNROLL>
__global__ void push_kernel(Ptrs p, int k_peers, int64_t nvec_per_peer, const float4* local) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int k = 0; k < k_peers; ++k) {
    float4* d = p.dst[k];
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < nvec_per_peer; i += stride) d[i] = local[i];
  }
}

// TMA bulk pull: one elected thread issues cp.async.bulk of CH bytes per peer per stage
__global__ void bulk_pull_kernel(Ptrs p, int k_peers, int64_t bytes_per_peer, int chunk, float4* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[4];
  const int stages = 4;
  unsigned char* buf = smem;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t chunks_per_peer = bytes_per_peer / chunk;
  const int64_t total = chunks_per_peer * k_peers;
  uint32_t phase[4] = {0, 0, 0, 0};
  float acc = 0.f;
  int64_t c0 = blockIdx.x;
  // prologue
  int issued = 0;
  for (int64_t c = c0; c < total; c += gridDim.x) {
    const int s = issued % stages;
    if (issued >= stages) {
      // wait for stage s to complete, consume
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(a), "r"(phase[s]));
      phase[s] ^= 1;
      acc += ((float*)(buf + (size_t)s * chunk))[threadIdx.x];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const int k = (int)(c / chunks_per_peer);
      const int64_t off = (c % chunks_per_peer) * chunk;
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + (size_t)s * chunk);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"((const char*)p.src[k] + off), "r"(chunk), "r"(a) : "memory");
    }
    ++issued;
  }
  for (int i = 0; i < stages && i < issued; ++i) {
    const int s = (issued + i) % stages;
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(a), "r"(phase[s]));
    phase[s] ^= 1;
  }
  if (acc == 12345.f) out[0].x = acc;
}

int main(int argc, char** argv) {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) { printf("{\"error\": \"need >= 2 GPUs\"}\n"); return 0; }
  const size_t bytes = 256ull << 20;  // per GPU buffer
  std::vector<float*> buf(ng), out(ng);
  for (int d = 0; d < ng; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < ng; ++e) if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaGetLastError();
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMalloc(&out[d], bytes));
    CK(cudaMemset(buf[d], 0, bytes));
    CK(cudaMemset(out[d], 0, bytes));
  }
  printf("{\"gpus\": %d, \"results\": [\n", ng);
  bool first = true;
  auto run = [&](const char* name, int k_peers, int grid, int block, int smem, auto launch) {
    std::vector<cudaEvent_t> a(ng), b(ng);
    for (int rep = 0; rep < 4; ++rep) {
      for (int d = 0; d < ng; ++d) {
        CK(cudaSetDevice(d));
        if (rep == 0) { CK(cudaEventCreate(&a[d])); CK(cudaEventCreate(&b[d])); }
        CK(cudaEventRecord(a[d]));
        launch(d);
        CK(cudaEventRecord(b[d]));
      }
      for (int d = 0; d < ng; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    }
    float worst = 0;
    for (int d = 0; d < ng; ++d) { float ms; CK(cudaEventElapsedTime(&ms, a[d], b[d])); if (ms > worst) worst = ms; }
    const double moved = (double)k_peers * (bytes / ng);  // bytes each GPU moved over NVLink
    printf("%s  {\"kernel\": \"%s\", \"peers\": %d, \"grid\": %d, \"block\": %d, \"us\": %.2f, \"GBps_per_gpu\": %.1f}\n",
           first ? "" : ",", name, k_peers, grid, block, worst * 1e3, moved / (worst * 1e-3) / 1e9);
    first = false;
  };
  for (int k_peers : {1, ng - 1}) {
    if (k_peers < 1) continue;
    const int64_t nvec = (bytes / ng) / 16;
    for (int grid : {148, 296, 592}) {
      for (int block : {256, 512}) {
        run("pull_cg_u4", k_peers, grid, block, 0, [&](int d) {
          Ptrs p{};
          for (int k = 0; k < k_peers; ++k) p.src[k] = (const float4*)buf[(d + 1 + k) % ng];
          pull_kernel<4, 1><<<grid, block>>>(p, k_peers, nvec, (float4*)out[d]);
        });
      }
    }
    run("pull_plain_u4", k_peers, 296, 512, 0, [&](int d) {
      Ptrs p{};
      for (int k = 0; k < k_peers; ++k) p.src[k] = (const float4*)buf[(d + 1 + k) % ng];
      pull_kernel<4, 0><<<296, 512>>>(p, k_peers, nvec, (float4*)out[d]);
    });
    run("pull_cg_u1", k_peers, 296, 512, 0, [&](int d) {
      Ptrs p{};
      for (int k = 0; k < k_peers; ++k) p.src[k] = (const float4*)buf[(d + 1 + k) % ng];
      pull_kernel<1, 1><<<296, 512>>>(p, k_peers, nvec, (float4*)out[d]);
    });
    run("pull_cg_u8", k_peers, 296, 512, 0, [&](int d) {
      Ptrs p{};
      for (int k = 0; k < k_peers; ++k) p.src[k] = (const float4*)buf[(d + 1 + k) % ng];
      pull_kernel<8, 1><<<296, 512>>>(p, k_peers, nvec, (float4*)out[d]);
    });
    for (int grid : {148, 296, 592}) {
      run("push", k_peers, grid, 512, 0, [&](int d) {
        Ptrs p{};
        for (int k = 0; k < k_peers; ++k) p.dst[k] = (float4*)out[(d + 1 + k) % ng] + (size_t)d * 0;  // same region ok
        push_kernel<1><<<grid, 512>>>(p, k_peers, nvec, (const float4*)buf[d]);
      });
    }
    for (int chunk : {8192, 16384, 32768}) {
      for (int grid : {148, 296}) {
        CK(cudaSetDevice(0));
        for (int d = 0; d < ng; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaFuncSetAttribute(bulk_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * chunk));
        }
        char name[64];
        snprintf(name, sizeof name, "bulk_pull_%dk", chunk / 1024);
        run(name, k_peers, grid, 256, 4 * chunk, [&](int d) {
          Ptrs p{};
          for (int k = 0; k < k_peers; ++k) p.src[k] = (const float4*)buf[(d + 1 + k) % ng];
          bulk_pull_kernel<<<grid, 256, 4 * chunk>>>(p, k_peers, (int64_t)(bytes / ng), chunk, (float4*)out[d]);
        });
      }
    }
  }
  printf("]}\n");
  return 0;
}
