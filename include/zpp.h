/*
 * zpp.h -- C ABI of the B200-native ZeRO++ communication-reduction hot path
 * (libzpp.so, sm_100a).
 *
 * The reference (zerosim, pure Python/numpy, /root/reference/pkg/src/zerosim)
 * has no FFI; its plugin point for this path is the codec object plus the
 * module-level functions re-exported from zerosim/__init__.py.  Each entry
 * point below replaces the compute of one of those reference functions; the
 * Python package paper_2306_10209_b200 binds them through ctypes and keeps the
 * reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every pointer is a device pointer unless
 *     stated otherwise; `stream` is a cudaStream_t (NULL = legacy stream).
 *   - All launches are asynchronous and stream-ordered.  The caller owns every
 *     buffer (the library allocates nothing on the hot path; only
 *     zpp_comm_create allocates the symmetric workspace).
 *   - Host-detectable errors (config, shapes) are returned synchronously.
 *     Device-detected conditions are OR-ed into *errflag (a device uint32):
 *       ZPP_FLAG_NONFINITE -> reference ValidationError (zs/quantizer.py:73-74)
 *       ZPP_FLAG_BADCODE   -> reference IntegrityError  (zs/quantizer.py:234-235)
 *       ZPP_FLAG_TIMEOUT   -> a peer never reached a device barrier
 *     errflag may be NULL (conditions are then not reported).
 *   - Wire format of one quantized tensor of n elements, block B, b bits:
 *       codes : ceil(n/B)*B*b/8 bytes, INT8 two's complement or INT4 two
 *               nibbles per byte, low nibble first (zs/quantizer.py:185-189),
 *               zero padding of the last block included;
 *       absmax: ceil(n/B) per-block max|x| as fp32 (inputs fp16/bf16/fp32:
 *               exact) or f64 (f64 inputs and fused requantization outputs).
 *     The reference scale is f64(absmax)/qmax, bit-exact (zpp_scales).
 */
#ifndef ZPP_H_
#define ZPP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes <-> zs/errors.py:9-30 */
enum {
  ZPP_OK = 0,
  ZPP_ERR_CONFIG = 1,     /* ConfigError     */
  ZPP_ERR_VALIDATION = 2, /* ValidationError */
  ZPP_ERR_INTEGRITY = 3,  /* IntegrityError  */
  ZPP_ERR_CUDA = 4,
  ZPP_ERR_COMM = 5
};

/* element types */
enum { ZPP_F32 = 0, ZPP_F16 = 1, ZPP_BF16 = 2, ZPP_F64 = 3 };

/* device error flag bits */
enum { ZPP_FLAG_NONFINITE = 1, ZPP_FLAG_BADCODE = 2, ZPP_FLAG_TIMEOUT = 4 };

int zpp_version(void);
const char* zpp_last_error(void);
int zpp_device_sm_count(void);

/* ---- codec ------------------------------------------------------------ */

/* K0  quantize(FlatTensor, QuantConfig)            zs/quantizer.py:204-228
 * x: n elements of dtype; absmax: fp32 for F32/F16/BF16 inputs, f64 for F64.
 * block = QuantConfig.block_size, or the effective full_tensor block
 * (zs/quantizer.py:179-182) computed by the caller. */
int zpp_quantize(const void* x, int dtype, int64_t n, int bits, int64_t block, void* codes, void* absmax,
                 void* errflag, void* stream);

/* K1  qgZ hop-1 encode of one stage                zs/collectives.py:509-518
 * grad: n elements (one rank's full gradient bucket); writes the send buffer
 * [j < X][c < Y][e < L] (L = n / (S*X*Y)) quantized in blocks of `block`
 * (L % block == 0).  reorder != 0 applies reorder_mapping's inverse
 * (zs/collectives.py:407-417, :498-499); reorder == 0 reproduces the
 * reference's reorder=False routing. */
int zpp_swizzle_quantize(const void* grad, int dtype, int64_t n, int X, int Y, int S, int stage, int reorder,
                         int bits, int64_t block, void* codes, void* absmax, void* errflag, void* stream);

/* K4  dequantize(QuantizedTensor)                  zs/quantizer.py:231-238
 * out: n elements of out_dtype, each the correctly rounded f64 code*scale. */
int zpp_dequantize(const void* codes, const void* absmax, int absmax_dtype, int64_t n, int bits, int64_t block,
                   void* out, int out_dtype, void* errflag, void* stream);

/* K4  gather-dequantize: the receive side of all_gather_qwz
 * (zs/collectives.py:264).  codes[s]/absmax[s] (host arrays of n_src device
 * pointers, local or NVLink peer) are decoded into out[s*shard_len ...].
 * rot staggers which source each warp starts with.  out_stride = elements
 * between consecutive sources' segments in out (0 = shard_len; larger strides
 * let a chunked caller gather piece k of every shard in place).  Optional hpZ
 * write-through: out elements [sec_lo, sec_lo+sec_len) are also written to
 * sec_out (NULL to skip). */
int zpp_gather_dequantize(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src,
                          int rot, int64_t shard_len, int bits, int64_t block, void* out, int out_dtype,
                          int64_t out_stride, void* sec_out, int64_t sec_lo, int64_t sec_len, void* errflag,
                          void* stream);

/* K3  BlockCodec.reduce_final                      zs/collectives.py:71-75
 * out[i] = post_scale * fold_{s ascending}(+0.0, code_s[i]*scale_s) in f64. */
int zpp_dequant_reduce(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
                       int bits, int64_t block, void* out, int out_dtype, double post_scale, void* errflag,
                       void* stream);

/* K2  fused_dequant_reduce_quant                   zs/quantizer.py:241-258
 * n_src inputs of n elements (in_bits/in_block) -> one tensor quantized with
 * out_bits/out_block; out_absmax is f64.  workspace (device) of
 * zpp_drq_workspace_bytes(n, out_block) bytes, may be NULL when that is 0. */
int zpp_dequant_reduce_quant(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src,
                             int64_t n, int in_bits, int64_t in_block, int out_bits, int64_t out_block,
                             void* out_codes, void* out_absmax, void* workspace, size_t workspace_bytes,
                             void* errflag, void* stream);
size_t zpp_drq_workspace_bytes(int64_t n, int64_t out_block);

/* QuantizedTensor.to_bytes on the device (replaces zs/quantizer.py:121-131):
 * writes the canonical wire layout -- 13-byte '<QBI' header (original_len,
 * bit_width, block_size), ceil(n/block) fp16 scales (RN-even of the f64 scale),
 * then the packed codes incl. padding -- into `out` (device, unaligned ok;
 * 13 + 2*n_blocks + code bytes long). */
int zpp_wire_pack(const void* codes, const void* absmax, int absmax_dtype, int64_t n, int bits, int64_t block,
                  void* out, void* stream);
/* QuantizedTensor.from_bytes payload on the device (zs/quantizer.py:133-149):
 * `raw` is the whole wire buffer (header already validated by the host);
 * writes the codes and an f64 absmax = fp16 scale * qmax (exact). */
int zpp_wire_unpack(const void* raw, int64_t n, int bits, int64_t block, void* codes, void* absmax_f64,
                    void* stream);

/* QuantizedTensor.scales: f64(absmax)/qmax, bit-exact (zs/quantizer.py:219) */
int zpp_scales(const void* absmax, int absmax_dtype, int64_t n_blocks, int bits, void* out_f64, void* stream);

/* ---- multi-GPU (one process per GPU, NVLink P2P over CUDA IPC) ---------- */

typedef struct zpp_comm* zpp_comm_t;
#define ZPP_IPC_HANDLE_BYTES 64

/* Allocates `sym_bytes` of device memory that every rank maps (symmetric
 * workspace) plus barrier flags.  group_size = GPUs per group (the
 * reference's gpus_per_node, zs/topology.py:31-52). */
int zpp_comm_create(int rank, int world, int group_size, size_t sym_bytes, zpp_comm_t* out);
/* this rank's IPC handle (ZPP_IPC_HANDLE_BYTES bytes, host memory) */
int zpp_comm_ipc_handle(zpp_comm_t comm, void* handle_out);
/* all ranks' handles, world * ZPP_IPC_HANDLE_BYTES bytes in rank order (host) */
int zpp_comm_open_peers(zpp_comm_t comm, const void* all_handles);
/* device address (in this process) of `rank`'s symmetric buffer */
void* zpp_comm_sym_ptr(zpp_comm_t comm, int rank);
size_t zpp_comm_sym_bytes(zpp_comm_t comm);
/* device barrier among ranks: scope 0 = world, 1 = my group, 2 = my cross set
 * (same local index in every group).  Bounded spin (timeout_ms). */
int zpp_comm_barrier(zpp_comm_t comm, int scope, int timeout_ms, void* errflag, void* stream);
/* After a barrier TIMEOUT (errflag bit 4) every data kernel sharing that flag
 * returns without touching its buffers.  Recovery: every rank synchronises
 * its device and passes a host barrier, then calls zpp_comm_reset (zeroes this
 * rank's barrier flag words, restarts the epochs and double-buffer phases),
 * clears errflag, and passes a second host barrier.  No reference
 * counterpart: the simulated fabric (zs/simnet.py) cannot time out. */
int zpp_comm_reset(zpp_comm_t comm);
/* Frees this rank's symmetric buffer.  Peers may still read it: call only
 * after every rank has synchronised and passed a host barrier. */
int zpp_comm_destroy(zpp_comm_t comm);
/* Stage tracer (diagnostics; not in the reference): while enabled, each qwZ /
 * qgZ call records timing events on its stream after every launch.
 * zpp_comm_trace_read waits for the last call's events and writes, per event,
 * the stage that had just finished (0 begin, 1 quantize, 2 barrier, 3 gather,
 * 4 K1, 5 K2, 6 K3) and the ms since the call began; returns the event count,
 * or -status on error. */
int zpp_comm_trace(zpp_comm_t comm, int enable);
int zpp_comm_trace_read(zpp_comm_t comm, int* ids, float* ms, int max);

/* qwZ all-gather, fused over NVLink (zs/collectives.py:244-282):
 * quantize this rank's shard into the symmetric buffer, world barrier, then
 * every rank decodes all W shards by peer loads straight into out
 * (W*shard_len elements; out_stride as in zpp_gather_dequantize).  Optional
 * hpZ write-through of out[sec_lo, sec_lo+sec_len) into sec_out. */
int zpp_qwz_allgather(zpp_comm_t comm, size_t sym_offset, const void* shard, int dtype, int64_t shard_len, int bits,
                      int64_t block, void* out, int out_dtype, int64_t out_stride, void* sec_out, int64_t sec_lo,
                      int64_t sec_len, void* errflag, void* stream);

/* qwZ all-gather of this layer with the next layer's quantization prefetched
 * (PAPER.md:611-618): as zpp_qwz_allgather, and when next_shard != NULL, K0 of
 * next_shard (next_len elements, same dtype and config) is launched on the
 * communicator's side stream into the next call's half of the symmetric
 * region, beside this call's NVLink gather.  The next call whose shard is
 * (next_shard, next_len) waits for that work instead of quantizing.
 * next_shard must stay unchanged until then.  Prefetch is skipped (the next
 * call quantizes as usual) when the layout would change or world == 1. */
int zpp_qwz_allgather_next(zpp_comm_t comm, size_t sym_offset, const void* shard, int dtype, int64_t shard_len,
                           int bits, int64_t block, void* out, int out_dtype, int64_t out_stride, void* sec_out,
                           int64_t sec_lo, int64_t sec_len, const void* next_shard, int64_t next_len, void* errflag,
                           void* stream);

/* hpZ secondary-partition all-gather inside the group over NVLink
 * (zs/collectives.py:202-241 with groups = PartitionSpec.groups()):
 * every rank's secondary shard (sec_len elements of elem_bytes) is held in
 * HBM at byte sym_offset of its symmetric buffer (written there by the qwZ
 * write-through, zs/engine.py:364-367); out receives the group's shards in
 * member order. */
int zpp_hpz_allgather(zpp_comm_t comm, size_t sym_offset, int64_t sec_len, int elem_bytes, void* out,
                      void* errflag, void* stream);

/* qgZ 2-hop quantized reduce-scatter over NVLink (zs/collectives.py:464-569):
 * grad: n elements; out: n/W elements (out_dtype), rank r's partition sum. */
int zpp_qgz_reduce_scatter(zpp_comm_t comm, size_t sym_offset, const void* grad, int dtype, int64_t n, int stages, int reorder,
                           int intra_bits, int64_t intra_block, int inter_bits, int64_t inter_block, void* out,
                           int out_dtype, void* errflag, void* stream);

/* qgZ over n_buckets consecutive buckets of n elements each (a gradient
 * stream cut into buckets, BASELINE configs[3]; zs/engine.py:455-506 reduces
 * a model's gradients this way): bucket b is one zpp_qgz_reduce_scatter of
 * grad[b*n, (b+1)*n) into out[b*n/W, (b+1)*n/W).  Same results as n_buckets
 * separate calls.  With one group (Y = 1) K1 of bucket b+1 runs on the
 * communicator's side stream beside the pulling K2 of bucket b; with a
 * second hop the buckets run back to back (measured faster).  No reference
 * counterpart beyond the per-bucket qgz_2hop (zs/collectives.py:464-569). */
int zpp_qgz_reduce_scatter_buckets(zpp_comm_t comm, size_t sym_offset, const void* grad, int dtype, int64_t n,
                                   int n_buckets, int stages, int reorder, int intra_bits, int64_t intra_block,
                                   int inter_bits, int64_t inter_block, void* out, int out_dtype, void* errflag,
                                   void* stream);

/* symmetric-workspace bytes each fused collective needs at its sym_offset
 * (double-buffered; 256-byte aligned regions) */
size_t zpp_qwz_sym_bytes(int64_t shard_len, int bits, int64_t block, int world);
size_t zpp_qgz_sym_bytes(int64_t n, int world, int stages, int intra_bits, int64_t intra_block, int inter_bits,
                         int64_t inter_block);
size_t zpp_hpz_sym_bytes(int64_t sec_len, int elem_bytes);

#ifdef __cplusplus
}
#endif
#endif /* ZPP_H_ */
