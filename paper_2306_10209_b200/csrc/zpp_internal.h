// Internal host-side declarations shared by the codec and comm translation units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "../../include/zpp.h"

namespace zpp {

// thread-local last error message + status
int fail(int status, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);

int sm_count();

struct AddrSpec {
  bool swizzle = false;
  int64_t n = 0;                // plain: valid input elements
  int64_t L = 0, part = 0, stage_off = 0;
  int X = 1, Y = 1, reorder = 1;
};

// launchers (validated arguments)
int launch_quantize(const void* x, int dtype, const AddrSpec& a, int64_t n_out, int bits, int64_t block,
                    uint8_t* codes, void* absmax, uint32_t* flag, cudaStream_t st);
// K1 fused with the qgZ hop-1 push: message j of the send buffer (msg_blocks
// blocks) goes to dst_codes[j] / dst_absmax[j] (fp32); tiles cycle through
// the messages starting at `first`.  *handled = false when
// the shape has no push path (the caller then quantizes locally).
int launch_quantize_push(const void* x, int dtype, const AddrSpec& a, int64_t n_out, int bits, int64_t block,
                         uint8_t* const* dst_codes, uint8_t* const* dst_absmax, int64_t msg_blocks, int first, int self_msg,
                         uint32_t* flag, cudaStream_t st, bool* handled);
int launch_quantize_deq(const void* x, int dtype, int64_t n, int bits, int64_t block, uint8_t* codes, void* absmax,
                        void* out, uint32_t* flag, cudaStream_t st, bool* handled);
int launch_gather_dequant(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src,
                          int rot, int64_t shard_len, int bits, int64_t block, void* out, int out_dtype,
                          void* sec_out, int64_t sec_lo, int64_t sec_len, uint32_t* flag, cudaStream_t st,
                          int64_t out_stride = 0);
int launch_dequant_reduce(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src,
                          int64_t n, int bits, int64_t block, void* out, int out_dtype, double post_scale,
                          uint32_t* flag, cudaStream_t st, bool validate = true);
int launch_drq(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
               int in_bits, int64_t in_block, int out_bits, int64_t out_block, uint8_t* out_codes,
               double* out_absmax, void* workspace, size_t ws_bytes, uint32_t* flag, cudaStream_t st,
               bool validate = true);
struct HopDst;  // zpp_kernels.cuh
int launch_drq_hop(const void* const* codes, const void* const* absmax, int n_src, int64_t n, int in_bits,
                   int64_t in_block, int out_bits, int64_t out_block, const HopDst& hop, uint32_t* flag,
                   cudaStream_t st, bool* handled);
int launch_drq_final(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
                     int in_bits, int64_t in_block, int out_bits, int64_t out_block, double* out_absmax, void* out,
                     int out_dtype, uint32_t* flag, cudaStream_t st, bool* handled);
// TMA-fed K2 / K3 for the communicator's qgZ hops (sources in symmetric,
// 256-byte padded regions).  *handled = false when the shape has no TMA path.
// final_out != nullptr: K2 writes the final partition (hop 2 is a self-send).
int launch_drq_tma(const void* const* codes, const void* const* absmax, int n_src, int64_t n, int in_bits,
                   int64_t in_block, int out_bits, int64_t out_block, uint8_t* out_codes, double* out_absmax,
                   void* final_out, int final_dtype, uint32_t* flag, cudaStream_t st, bool* handled);
int launch_dr_tma(const void* const* codes, const void* const* absmax_f64, int n_src, int64_t n, int bits,
                  int64_t block, void* out, int out_dtype, uint32_t* flag, cudaStream_t st, bool* handled);
size_t drq_workspace_bytes(int64_t n, int64_t out_block);
bool drq_has_reg_path(int64_t out_block);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t code_bytes(int64_t n, int bits, int64_t block) {
  return ceil_div(n, block) * block * bits / 8;
}

}  // namespace zpp
