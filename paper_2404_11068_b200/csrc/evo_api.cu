// evo_api.cu — the C ABI (include/evo_attn.h): validation, TMA descriptors, workspace carving,
// kernel dispatch.  No torch types, no allocation on the hot path, no CPU fallback.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "evo_attn.h"
#include "evo_kernels.cuh"

namespace {

thread_local std::string g_detail;
}  // namespace
namespace evo {
void set_error_detail(const char* msg) { g_detail = msg; }
}  // namespace evo
namespace {
thread_local int g_launches = 0;
// SM count of the current device: fixes the batch chunking of the dbias partials (one CTA per SM
// in the fused backward), so the workspace is a function of the descriptor and the device.
// Queried once per device (148 on B200; no device -> 148, so the CPU-side size queries agree).
int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    (void)cudaGetLastError();
    return 148;
  }
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      (void)cudaGetLastError();
      n = 148;
    }
    cache[dev] = n;
  }
  return cache[dev];
}

evo_status_t fail(evo_status_t s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
evo_status_t fail(evo_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_detail = buf;
  return s;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

inline int esize(const evo_attn_desc_t* d) { return d->dtype == EVO_BF16 ? 2 : 4; }
inline int dpad(int D) { return D < 16 ? 16 : D; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

evo_status_t check_strides(const char* name, const int64_t* s, int64_t e0, int64_t e1, int64_t e2,
                           int es) {
  const int64_t ext[3] = {e0, e1, e2};
  for (int i = 0; i < 3; ++i) {
    if (ext[i] <= 1) continue;
    if (s[i] < 1) return fail(EVO_E_SHAPE, "%s_str[%d] = %lld must be >= 1", name, i, (long long)s[i]);
    if ((s[i] * es) % 16 != 0)
      return fail(EVO_E_ALIGN, "%s_str[%d] = %lld elements is not a multiple of 16 bytes", name,
                  i, (long long)s[i]);
  }
  return EVO_OK;
}

int bias_mode(const evo_attn_desc_t* d) {  // 0 none, 1 k-contiguous, 2 q-contiguous
  if (d->bias_kind == EVO_BIAS_NONE) return 0;
  if (d->bias_str[3] == 1 || d->Lk <= 1) return 1;
  return 2;
}

// Tensor map over a logical [B][H][L][D] tensor with element strides (b, h, l), unit d.
bool make_x_map(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int es, int64_t B,
                int64_t H, int64_t L, int D, const int64_t str[3], int box_rows = 128,
                int box_cols = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  const int DP = dpad(D);
  const int64_t ext[3] = {B, H, L};
  cuuint64_t sb[3];
  int64_t span = (int64_t)D * es;
  for (int i = 2; i >= 0; --i) {  // l, h, b
    int64_t s = str[i] * es;
    if (ext[i] <= 1 || s <= 0) s = ((span + 15) / 16) * 16;
    sb[i] = (cuuint64_t)s;
    span = std::max<int64_t>(span, s * std::max<int64_t>(ext[i], 1));
  }
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)std::max<int64_t>(L, 1),
                        (cuuint64_t)std::max<int64_t>(H, 1), (cuuint64_t)std::max<int64_t>(B, 1)};
  cuuint64_t strides[3] = {sb[2], sb[1], sb[0]};
  const int bc = box_cols > 0 ? box_cols : DP;
  cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const int rowb = bc * es;
  CUtensorMapSwizzle sw = rowb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                     : (rowb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_128B);
  return enc(m, dt, 4, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Bias tile map: rows = non-contiguous index, cols = contiguous index; box 64 cols x 128 rows.
bool make_bias_map(CUtensorMap* m, const evo_attn_desc_t* d, const void* bias,
                   int box_rows = 128) {
  auto enc = get_encode();
  if (!enc) return false;
  const int mode = bias_mode(d);
  const int64_t Bb = d->bias_kind == EVO_BIAS_PER_BATCH ? d->B : 1;
  const int64_t c_ext = mode == 1 ? d->Lk : d->Lq, r_ext = mode == 1 ? d->Lq : d->Lk;
  const int64_t r_str = mode == 1 ? d->bias_str[2] : d->bias_str[3];
  const int64_t ext[3] = {Bb, d->H, r_ext};
  const int64_t str[3] = {d->bias_str[0], d->bias_str[1], r_str};
  cuuint64_t sb[3];
  int64_t span = c_ext * 2;
  for (int i = 2; i >= 0; --i) {
    int64_t s = str[i] * 2;
    if (ext[i] <= 1 || s <= 0) s = ((span + 15) / 16) * 16;
    sb[i] = (cuuint64_t)s;
    span = std::max<int64_t>(span, s * std::max<int64_t>(ext[i], 1));
  }
  cuuint64_t dims[4] = {(cuuint64_t)std::max<int64_t>(c_ext, 1),
                        (cuuint64_t)std::max<int64_t>(r_ext, 1), (cuuint64_t)d->H,
                        (cuuint64_t)std::max<int64_t>(Bb, 1)};
  cuuint64_t strides[3] = {sb[2], sb[1], sb[0]};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(bias), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct WsLayout {
  size_t lse2 = 0, dvec = 0, da = 0, dqacc = 0, partial = 0, total = 0;
  int nchunks = 1, chunk = 1;
  bool fused = false;
};
// Single-pass backward (evo_bwd_pb.cu / evo_bwd_nb.cu) for bf16 with a shared bias (Lq <= 384)
// or none
bool use_fused_bwd(const evo_attn_desc_t* d) {
  if (d->dtype != EVO_BF16 || d->bias_kind == EVO_BIAS_PER_BATCH) return false;
  const int Lq_pad = ((d->Lq + 127) / 128) * 128;
  return evo::bwd_fused_supported(dpad(d->D), Lq_pad, d->bias_kind != EVO_BIAS_NONE);
}
// dQ over several key tiles.  Determinism (bitwise-repeatable backward): with
// exactly two key tiles both reduce-add (TMA .add at L2) into ONE fp32 accumulator that bwd_pre
// zero-fills, and 0 + a + b = 0 + b + a exactly, so the order of the two adds cannot change a
// bit; with three or more key tiles fp32 addition is not associative, so every key tile stores
// its own fp32 part and dq_convert sums the parts in key-tile order 0, 1, ..., nk-1.
// No bias, several key tiles, enough (b, h) rows to fill the SMs: the no-bias kernel walks all
// key tiles of a row inside one CTA and accumulates dQ in TMEM in key-tile order (deterministic,
// no fp32 parts, no dq_convert)
bool use_nb_kloop(const evo_attn_desc_t* d) {
  const int nq = (int)((d->Lq + 127) / 128), nk = (int)((d->Lk + 127) / 128);
  return use_fused_bwd(d) && d->bias_kind == EVO_BIAS_NONE && nk > 1 &&
         evo::bwd_nb_kloop_fits(dpad(d->D), nq) && d->B * d->H >= num_sms();
}
// Shared bias, Lq <= 256, exactly two key tiles (the bias modules at N_res / N_seq = 256): the
// pair-bias kernel runs the two key tiles of a (h, chunk) as a 2-CTA cluster and sums dQ on
// chip (dQ_0 + dQ_1 in that order: deterministic, no fp32 accumulator, no dq_convert)
bool use_dq_pair(const evo_attn_desc_t* d) {
  const int nk = (int)((d->Lk + 127) / 128), Lq_pad = (int)((d->Lq + 127) / 128) * 128;
  // rank 0/1 store their dq rows with 16-B vector stores: D % 8 == 0 and 16-B aligned rows
  const bool vec = d->D % 8 == 0 && d->q_str[0] % 8 == 0 && d->q_str[1] % 8 == 0 && d->q_str[2] % 8 == 0;
  return use_fused_bwd(d) && d->bias_kind == EVO_BIAS_SHARED && Lq_pad <= 256 && nk == 2 && vec;
}
bool use_dq_reduce(const evo_attn_desc_t* d) {
  const int64_t nk = (d->Lk + 127) / 128;
  const int64_t pre_vec = d->B * d->H * ((d->Lq + 127) / 128 * 128) * (d->D / 8);
  return use_fused_bwd(d) && !use_nb_kloop(d) && !use_dq_pair(d) && nk == 2 && d->D % 8 == 0 &&
         pre_vec < ((int64_t)1 << 31);  // the conditions of bwd_pre's vectorised path
}
inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

WsLayout ws_layout(const evo_attn_desc_t* d) {
  WsLayout w;
  const int64_t nq = (d->Lq + 127) / 128, nk = (d->Lk + 127) / 128;
  const int64_t Lq_pad = nq * 128, Lk_pad = nk * 128;
  const int64_t rows = d->B * d->H;
  size_t off = 0;
  w.lse2 = off; off = al256(off + (size_t)rows * Lq_pad * 4);
  w.dvec = off; off = al256(off + (size_t)rows * Lq_pad * 4);
  if (d->has_gate) { w.da = off; off = al256(off + (size_t)rows * d->Lq * d->D * esize(d)); }
  if (d->dtype == EVO_BF16 && nk > 1 && !use_nb_kloop(d) && !use_dq_pair(d)) {
    // one fp32 accumulator (nk == 2, reduce-add) or one fp32 part per key tile (use_dq_reduce)
    w.dqacc = off;
    const int64_t parts = use_dq_reduce(d) ? 1 : nk;
    off = al256(off + (size_t)parts * rows * d->Lq * d->D * 4);
  }
  w.fused = use_fused_bwd(d);
  if (d->dtype == EVO_BF16 && d->bias_kind != EVO_BIAS_NONE && d->B > 0) {
    int64_t nch, chunk;
    if (w.fused) {
      int ch = 1;
      nch = evo::bwd_fused_nchunks((int)d->B, d->H, (int)nk, num_sms(), &ch);
      chunk = ch;
    } else {
      const int64_t tiles = (int64_t)d->H * nq * nk;
      nch = (2 * num_sms() + tiles - 1) / std::max<int64_t>(tiles, 1);
      nch = std::max<int64_t>(1, std::min<int64_t>(nch, d->B));
      chunk = (d->B + nch - 1) / nch;
      nch = (d->B + chunk - 1) / chunk;
    }
    w.nchunks = (int)nch;
    w.chunk = (int)chunk;
    const int64_t parts = d->bias_kind == EVO_BIAS_PER_BATCH ? d->B : nch;
    w.partial = off;
    off = al256(off + (size_t)parts * d->H * Lq_pad * Lk_pad * 4);
  }
  w.total = off;
  return w;
}

evo_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(EVO_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------------ optional kernel tracing
struct Trace {
  cudaEvent_t* ev = nullptr;
  int cap = 0, n = 0;
  const char* labels[4096];
};
thread_local Trace g_trace;
inline void trace_begin(cudaStream_t st, const char* label) {
  Trace& t = g_trace;
  if (!t.ev || 2 * t.n + 1 >= t.cap || t.n >= 4096) return;
  t.labels[t.n] = label;
  if (cudaEventRecord(t.ev[2 * t.n], st) != cudaSuccess) {
    (void)cudaGetLastError();  // a bad trace event must not poison the kernel launch
    t.ev = nullptr;
  }
}
inline void trace_end(cudaStream_t st) {
  Trace& t = g_trace;
  if (!t.ev || 2 * t.n + 1 >= t.cap || t.n >= 4096) return;
  if (cudaEventRecord(t.ev[2 * t.n + 1], st) != cudaSuccess) {
    (void)cudaGetLastError();
    t.ev = nullptr;
    return;
  }
  ++t.n;
}
// Per-host-thread side stream (+ fork/join events) of the current device: the two independent
// tails of the fused backward (dq parts -> bf16, dbias partials -> dbias) run concurrently, the
// dbias reduce forked off the caller's stream and joined back before the call returns (so the
// call stays stream-ordered; fork/join by events is also what CUDA-graph capture records).
struct SideStream {
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream* side_stream() {
  thread_local SideStream ss;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (ss.dev != dev) {
    SideStream n;
    n.dev = dev;
    if (cudaStreamCreateWithFlags(&n.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&n.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&n.join, cudaEventDisableTiming) != cudaSuccess) {
      (void)cudaGetLastError();
      return nullptr;  // callers fall back to running both tails on the caller's stream
    }
    ss = n;  // (a previous device's stream/events are left to the process teardown)
  }
  return &ss;
}

// launch wrapper: bracket one kernel launch with trace events
template <class F>
inline cudaError_t traced(cudaStream_t st, const char* label, F&& f) {
  trace_begin(st, label);
  cudaError_t e = f();
  trace_end(st);
  return e;
}

}  // namespace

extern "C" {

int evo_abi_version(void) { return EVO_ATTN_ABI_VERSION; }

int evo_trace_enable(void** events, int capacity) {
  if (capacity < 0) return EVO_E_INVALID;
  g_trace.ev = reinterpret_cast<cudaEvent_t*>(events);
  g_trace.cap = events ? capacity : 0;
  g_trace.n = 0;
  return EVO_OK;
}
int evo_trace_count(void) { return g_trace.n; }
const char* evo_trace_label(int i) {
  return (i >= 0 && i < g_trace.n) ? g_trace.labels[i] : nullptr;
}
int evo_last_launch_count(void) { return g_launches; }
const char* evo_last_error_detail(void) { return g_detail.c_str(); }

const char* evo_status_string(evo_status_t s) {
  switch (s) {
    case EVO_OK: return "EVO_OK";
    case EVO_E_INVALID: return "EVO_E_INVALID";
    case EVO_E_SHAPE: return "EVO_E_SHAPE";
    case EVO_E_ALIGN: return "EVO_E_ALIGN";
    case EVO_E_UNSUPPORTED: return "EVO_E_UNSUPPORTED";
    case EVO_E_WORKSPACE: return "EVO_E_WORKSPACE";
    case EVO_E_CUDA: return "EVO_E_CUDA";
  }
  return "EVO_E_UNKNOWN";
}

evo_status_t evo_attn_validate(const evo_attn_desc_t* d) {
  g_detail.clear();
  if (!d) return fail(EVO_E_INVALID, "descriptor is NULL");
  if (d->dtype != EVO_BF16 && d->dtype != EVO_F32) return fail(EVO_E_INVALID, "dtype %d", d->dtype);
  if (!(d->scale > 0.f) || !std::isfinite(d->scale))
    return fail(EVO_E_INVALID, "scale must be finite and > 0");
  if (d->B < 0 || d->H < 1 || d->Lq < 0 || d->Lk < 0)
    return fail(EVO_E_SHAPE, "B=%lld H=%d Lq=%d Lk=%d", (long long)d->B, d->H, d->Lq, d->Lk);
  if (d->D != 8 && d->D != 16 && d->D != 32 && d->D != 64)
    return fail(EVO_E_UNSUPPORTED, "head dim D=%d not in {8,16,32,64}", d->D);
  if (d->Lk > evo::kMaxLk) return fail(EVO_E_UNSUPPORTED, "Lk=%d > %d", d->Lk, evo::kMaxLk);
  if (d->bias_kind < 0 || d->bias_kind > 2) return fail(EVO_E_INVALID, "bias_kind %d", d->bias_kind);
  if ((d->has_mask != 0 && d->has_mask != 1) || (d->has_gate != 0 && d->has_gate != 1))
    return fail(EVO_E_INVALID, "has_mask / has_gate must be 0 or 1");
  const long long units = (long long)d->B * d->H * ((d->Lq + 127) / 128 + (d->Lk + 127) / 128);
  if (units >= (1ll << 31)) return fail(EVO_E_UNSUPPORTED, "problem too large for one launch");
  const int es = esize(d);
  evo_status_t s;
  if ((s = check_strides("q", d->q_str, d->B, d->H, d->Lq, es))) return s;
  if ((s = check_strides("k", d->k_str, d->B, d->H, d->Lk, es))) return s;
  if ((s = check_strides("v", d->v_str, d->B, d->H, d->Lk, es))) return s;
  if ((s = check_strides("o", d->o_str, d->B, d->H, d->Lq, es))) return s;
  if (d->has_gate && (s = check_strides("g", d->g_str, d->B, d->H, d->Lq, es))) return s;
  if (d->bias_kind != EVO_BIAS_NONE) {
    const bool kc = d->bias_str[3] == 1 || d->Lk <= 1, qc = d->bias_str[2] == 1 || d->Lq <= 1;
    if (!kc && !qc)
      return fail(EVO_E_UNSUPPORTED, "bias needs a unit stride along q or k (got q=%lld k=%lld)",
                  (long long)d->bias_str[2], (long long)d->bias_str[3]);
    const int mode = bias_mode(d);
    const int64_t rs = mode == 1 ? d->bias_str[2] : d->bias_str[3];
    const int64_t rext = mode == 1 ? d->Lq : d->Lk;
    const int64_t bs[3] = {d->bias_str[0], d->bias_str[1], rs};
    const int64_t bb = d->bias_kind == EVO_BIAS_PER_BATCH ? d->B : 1;
    if ((s = check_strides("bias", bs, bb, d->H, rext, es))) return s;
  }
  return EVO_OK;
}

size_t evo_attn_bwd_workspace_bytes(const evo_attn_desc_t* d) {
  if (evo_attn_validate(d) != EVO_OK) return 0;
  return ws_layout(d).total;
}

evo_status_t evo_attn_fwd(const evo_attn_desc_t* d, const void* q, const void* k, const void* v,
                          const void* bias, const uint8_t* mask, const void* g, void* o,
                          float* lse, void* stream) {
  g_launches = 0;
  evo_status_t s = evo_attn_validate(d);
  if (s) return s;
  if (!q || !k || !v || !o || !lse) return fail(EVO_E_INVALID, "q, k, v, o and lse are required");
  if ((bias != nullptr) != (d->bias_kind != EVO_BIAS_NONE))
    return fail(EVO_E_INVALID, "bias pointer must be non-NULL iff bias_kind != NONE");
  if ((mask != nullptr) != (d->has_mask != 0))
    return fail(EVO_E_INVALID, "mask pointer must be non-NULL iff has_mask");
  if ((g != nullptr) != (d->has_gate != 0))
    return fail(EVO_E_INVALID, "g pointer must be non-NULL iff has_gate");
  for (const void* p : {q, k, v, (const void*)o, (const void*)lse, bias, g})
    if (p && !aligned16(p)) return fail(EVO_E_ALIGN, "a tensor pointer is not 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (d->B == 0 || d->Lq == 0) return EVO_OK;
  if (d->Lk == 0) {
    cudaError_t e = evo::launch_fill_empty(lse, d->B * d->H * (int64_t)d->Lq, o, d->dtype, (int)d->B,
                                           d->H, d->Lq, d->D, d->o_str[0], d->o_str[1], d->o_str[2], st);
    g_launches = 1;
    return e == cudaSuccess ? EVO_OK : cuda_fail(e, "fill_empty");
  }
  if (d->dtype == EVO_F32) {
    evo::F32Args a{};
    a.B = (int)d->B; a.H = d->H; a.Lq = d->Lq; a.Lk = d->Lk; a.D = d->D; a.scale = d->scale;
    a.q = (const float*)q; a.k = (const float*)k; a.v = (const float*)v; a.g = (const float*)g;
    a.bias = (const float*)bias;
    a.q_sb = d->q_str[0]; a.q_sh = d->q_str[1]; a.q_sl = d->q_str[2];
    a.k_sb = d->k_str[0]; a.k_sh = d->k_str[1]; a.k_sl = d->k_str[2];
    a.v_sb = d->v_str[0]; a.v_sh = d->v_str[1]; a.v_sl = d->v_str[2];
    a.g_sb = d->g_str[0]; a.g_sh = d->g_str[1]; a.g_sl = d->g_str[2];
    a.bias_kind = d->bias_kind;
    a.b_sb = d->bias_str[0]; a.b_sh = d->bias_str[1]; a.b_sq = d->bias_str[2]; a.b_sk = d->bias_str[3];
    a.mask = mask; a.mask_s0 = d->mask_str[0]; a.mask_s1 = d->mask_str[1];
    a.o = (float*)o; a.o_sb = d->o_str[0]; a.o_sh = d->o_str[1]; a.o_sl = d->o_str[2];
    a.lse = lse;
    cudaError_t e = traced(st, "fwd_f32", [&] { return evo::launch_fwd_f32(a, st); });
    g_launches = 1;
    return e == cudaSuccess ? EVO_OK : cuda_fail(e, "fwd_f32");
  }
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int bm = bias_mode(d);
  evo::FwdOccLaunch O;
  memset(&O, 0, sizeof(O));
  if (!make_x_map(&O.tm_k, k, dt, 2, d->B, d->H, d->Lk, d->D, d->k_str, 64) ||
      !make_x_map(&O.tm_v, v, dt, 2, d->B, d->H, d->Lk, d->D, d->v_str, 64) ||
      (bm && !make_bias_map(&O.tm_b, d, bias, bm == 1 ? 128 : 64)))
    return fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed for k/v/bias");
  evo::FwdArgs& a = O.args;
  a.B = (int)d->B; a.H = d->H; a.Lq = d->Lq; a.Lk = d->Lk; a.D = d->D;
  a.scale = d->scale;
  a.scale_log2 = d->scale * evo::kLog2e;
  a.bias_batched = d->bias_kind == EVO_BIAS_PER_BATCH;
  a.mask = mask; a.mask_s0 = d->mask_str[0]; a.mask_s1 = d->mask_str[1];
  a.g = (const __nv_bfloat16*)g; a.g_sb = d->g_str[0]; a.g_sh = d->g_str[1]; a.g_sl = d->g_str[2];
  a.o = (__nv_bfloat16*)o; a.o_sb = d->o_str[0]; a.o_sh = d->o_str[1]; a.o_sl = d->o_str[2];
  a.lse = lse;
  O.q = (const __nv_bfloat16*)q;
  O.q_sb = d->q_str[0]; O.q_sh = d->q_str[1]; O.q_sl = d->q_str[2];
  cudaError_t e = traced(st, "fwd_bf16", [&] { return evo::launch_fwd_occ_bf16(O, dpad(d->D), bm, st); });
  g_launches = 1;
  return e == cudaSuccess ? EVO_OK : cuda_fail(e, "fwd_bf16");
}

evo_status_t evo_attn_bwd(const evo_attn_desc_t* d, const void* q, const void* k, const void* v,
                          const void* bias, const uint8_t* mask, const void* g, const void* o,
                          const float* lse, const void* dout, void* dq, void* dk, void* dv,
                          void* dg, float* dbias, void* workspace, size_t workspace_bytes,
                          void* stream) {
  g_launches = 0;
  evo_status_t s = evo_attn_validate(d);
  if (s) return s;
  if (!q || !k || !v || !o || !lse || !dout || !dq || !dk || !dv)
    return fail(EVO_E_INVALID, "q, k, v, o, lse, dout, dq, dk, dv are required");
  if ((bias != nullptr) != (d->bias_kind != EVO_BIAS_NONE) ||
      (dbias != nullptr) != (d->bias_kind != EVO_BIAS_NONE))
    return fail(EVO_E_INVALID, "bias / dbias must be non-NULL iff bias_kind != NONE");
  if ((mask != nullptr) != (d->has_mask != 0))
    return fail(EVO_E_INVALID, "mask pointer must be non-NULL iff has_mask");
  if ((g != nullptr) != (d->has_gate != 0) || (dg != nullptr) != (d->has_gate != 0))
    return fail(EVO_E_INVALID, "g / dg must be non-NULL iff has_gate");
  for (const void* p : {q, k, v, o, (const void*)lse, dout, (const void*)dq, (const void*)dk,
                        (const void*)dv, (const void*)dg, bias, g, (const void*)dbias, (const void*)workspace})
    if (p && !aligned16(p)) return fail(EVO_E_ALIGN, "a tensor pointer is not 16-byte aligned");
  const WsLayout W = ws_layout(d);
  if (W.total > 0 && (!workspace || workspace_bytes < W.total))
    return fail(EVO_E_WORKSPACE, "workspace needs %zu bytes, got %zu", W.total, workspace_bytes);
  if (d->B == 0 || d->Lq == 0 || d->Lk == 0)
    return fail(EVO_E_UNSUPPORTED, "backward of an empty problem (B, Lq or Lk == 0)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  float* lse2 = reinterpret_cast<float*>(ws + W.lse2);
  float* dvec = reinterpret_cast<float*>(ws + W.dvec);
  void* dA = d->has_gate ? (void*)(ws + W.da) : nullptr;
  const int nk = (d->Lk + 127) / 128;
  int nl = 0;
  cudaError_t e;

  evo::BwdPreArgs pa{};
  pa.B = (int)d->B; pa.H = d->H; pa.Lq = d->Lq; pa.D = d->D;
  pa.o = o; pa.dout = dout; pa.o_sb = d->o_str[0]; pa.o_sh = d->o_str[1]; pa.o_sl = d->o_str[2];
  pa.g = g; pa.g_sb = d->g_str[0]; pa.g_sh = d->g_str[1]; pa.g_sl = d->g_str[2]; pa.dg = dg;
  pa.lse = lse; pa.lse2 = lse2; pa.Dvec = dvec; pa.dA = dA;
  pa.negate = W.fused ? 1 : 0;
  // dA workspace: dense, in the (h, l) order of o's strides so bwd_pre's accesses coalesce
  const bool o_hfast = d->o_str[1] < d->o_str[2];
  const int64_t da_str[3] = {(int64_t)d->H * d->Lq * d->D, o_hfast ? d->D : (int64_t)d->Lq * d->D,
                             o_hfast ? (int64_t)d->H * d->D : d->D};
  pa.a_sb = da_str[0]; pa.a_sh = da_str[1]; pa.a_sl = da_str[2];
  // dQ over two key tiles: the fused backward reduce-adds (TMA .add, performed at L2) both key
  // tiles' fp32 dQ into ONE accumulator that the vectorised bwd_pre zero-fills on its way — one
  // fp32 part read by dq_convert instead of two; see use_dq_reduce for determinism
  const bool dq_red = use_dq_reduce(d);
  if (dq_red) {  // bwd_pre zero-fills the accumulator in the layout of the dQ parts
    const bool qh = d->q_str[1] < d->q_str[2];
    pa.zacc = reinterpret_cast<float*>(ws + W.dqacc);
    pa.z_sb = (int64_t)d->H * d->Lq * d->D;
    pa.z_sh = qh ? d->D : (int64_t)d->Lq * d->D;
    pa.z_sl = qh ? (int64_t)d->H * d->D : d->D;
  }
  if ((e = traced(st, "bwd_pre", [&] { return evo::launch_bwd_pre(pa, d->dtype == EVO_F32, st); })) != cudaSuccess) return cuda_fail(e, "bwd_pre");
  ++nl;
  // dA operand: workspace [B,H,Lq,D] contiguous, or dout itself when there is no gate
  const void* dA_ptr = d->has_gate ? dA : dout;
  const int64_t* dA_str = d->has_gate ? da_str : d->o_str;

  if (d->dtype == EVO_F32) {
    evo::F32Args a{};
    a.B = (int)d->B; a.H = d->H; a.Lq = d->Lq; a.Lk = d->Lk; a.D = d->D; a.scale = d->scale;
    a.q = (const float*)q; a.k = (const float*)k; a.v = (const float*)v; a.g = (const float*)g;
    a.bias = (const float*)bias;
    a.q_sb = d->q_str[0]; a.q_sh = d->q_str[1]; a.q_sl = d->q_str[2];
    a.k_sb = d->k_str[0]; a.k_sh = d->k_str[1]; a.k_sl = d->k_str[2];
    a.v_sb = d->v_str[0]; a.v_sh = d->v_str[1]; a.v_sl = d->v_str[2];
    a.bias_kind = d->bias_kind;
    a.b_sb = d->bias_str[0]; a.b_sh = d->bias_str[1]; a.b_sq = d->bias_str[2]; a.b_sk = d->bias_str[3];
    a.mask = mask; a.mask_s0 = d->mask_str[0]; a.mask_s1 = d->mask_str[1];
    a.dA = (const float*)dA_ptr; a.a_sb = dA_str[0]; a.a_sh = dA_str[1]; a.a_sl = dA_str[2];
    a.lse_in = lse; a.Dvec = dvec;
    a.dq = (float*)dq; a.dk = (float*)dk; a.dv = (float*)dv; a.dbias = dbias;
    e = traced(st, "bwd_f32", [&] { return evo::launch_bwd_f32(a, st, &nl); });
    g_launches = nl;
    return e == cudaSuccess ? EVO_OK : cuda_fail(e, "bwd_f32");
  }

  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUtensorMap tq, tk, tv, tda, tb;
  memset(&tb, 0, sizeof(tb));
  if (!make_x_map(&tq, q, dt, 2, d->B, d->H, d->Lq, d->D, d->q_str) ||
      !make_x_map(&tk, k, dt, 2, d->B, d->H, d->Lk, d->D, d->k_str) ||
      !make_x_map(&tv, v, dt, 2, d->B, d->H, d->Lk, d->D, d->v_str) ||
      !make_x_map(&tda, dA_ptr, dt, 2, d->B, d->H, d->Lq, d->D, dA_str))
    return fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed for q/k/v/dA");
  const int bm = bias_mode(d);
  if (bm && !make_bias_map(&tb, d, bias)) return fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed for bias");

  const bool kloop = use_nb_kloop(d), dq_pair = use_dq_pair(d);
  float* dqacc = nk > 1 && !kloop && !dq_pair ? reinterpret_cast<float*>(ws + W.dqacc) : nullptr;
  if (W.fused) {
    evo::BwdFusedLaunch F;
    F.tm_q = tq; F.tm_k = tk; F.tm_v = tv; F.tm_da = tda;
    // output maps of the dK/dV drains (bf16, k/v strides); the dQ parts (more than one key
    // tile) are fp32, dense, in dq's (h, l) order (dq_convert reads them coalesced that way)
    const bool q_hfast = d->q_str[1] < d->q_str[2];
    const int64_t part_str[3] = {(int64_t)d->H * d->Lq * d->D,
                                 q_hfast ? d->D : (int64_t)d->Lq * d->D,
                                 q_hfast ? (int64_t)d->H * d->D : d->D};
    // 32-row boxes: each compute warp stores its own TMEM lane quarter
    if (!make_x_map(&F.tm_dk, dk, dt, 2, d->B, d->H, d->Lk, d->D, d->k_str, 32) ||
        !make_x_map(&F.tm_dv, dv, dt, 2, d->B, d->H, d->Lk, d->D, d->v_str, 32) ||
        !(!dqacc ? make_x_map(&F.tm_dq, dq, dt, 2, d->B, d->H, d->Lq, d->D, d->q_str, 32)
                  : make_x_map(&F.tm_dq, dqacc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                               (int64_t)nk * d->B, d->H, d->Lq, d->D, part_str, 32,
                               std::min(dpad(d->D), 32))))
      return fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed for the output maps");
    evo::BwdFusedArgs& fa = F.args;
    memset(&fa, 0, sizeof(fa));
    fa.B = (int)d->B; fa.H = d->H; fa.Lq = d->Lq; fa.Lk = d->Lk; fa.D = d->D;
    fa.scale = d->scale; fa.scale_log2 = d->scale * evo::kLog2e;
    // same chunking as the workspace's dbias partials (ws_layout)
    fa.nchunks = evo::bwd_fused_nchunks((int)d->B, d->H, kloop ? 1 : nk, num_sms(), &fa.chunk);
    fa.kloop = kloop ? 1 : 0;
    fa.dq_pair = dq_pair ? 1 : 0;
    fa.bias = (const __nv_bfloat16*)bias;
    fa.b_sh = d->bias_str[1]; fa.b_sq = d->bias_str[2]; fa.b_sk = d->bias_str[3];
    fa.mask = mask; fa.mask_s0 = d->mask_str[0]; fa.mask_s1 = d->mask_str[1];
    fa.lse2 = lse2; fa.Dvec = dvec;
    fa.dk = (__nv_bfloat16*)dk; fa.k_sb = d->k_str[0]; fa.k_sh = d->k_str[1]; fa.k_sl = d->k_str[2];
    fa.dv = (__nv_bfloat16*)dv; fa.v_sb = d->v_str[0]; fa.v_sh = d->v_str[1]; fa.v_sl = d->v_str[2];
    fa.dq = (__nv_bfloat16*)dq; fa.q_sb = d->q_str[0]; fa.q_sh = d->q_str[1]; fa.q_sl = d->q_str[2];
    fa.dq_acc = dqacc;
    fa.p_part = (int64_t)d->B * d->H * d->Lq * d->D;
    fa.p_sb = part_str[0]; fa.p_sh = part_str[1]; fa.p_sl = part_str[2];
    fa.dq_reduce = dq_red ? 1 : 0;
    fa.bmode = bm;
    memset(&F.tm_b, 0, sizeof(F.tm_b));
    // 256 < Lq <= 384 with a bias ("big"): the k-contiguous biasᵀ prologue stages 128 queries
    // at a time, and a Σ-only second pass covers the query tile beyond 256
    const bool big = bm && ((d->Lq + 127) / 128) * 128 > 256;
    if (bm && !make_bias_map(&F.tm_b, d, bias, bm == 1 ? (big ? 128 : 256) : 128))
      return fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed for the fused backward's bias map");
    fa.partial = bm ? reinterpret_cast<float*>(ws + W.partial) : nullptr;
    fa.t0 = 0;
    fa.sigma_only = 0;
    if ((e = traced(st, "bwd_fused", [&] {
           // bias: 64-query hand-offs (256 < Lq <= 384: Σ of the first 256 queries, the Σ-only
           // pass below adds the last tile's); no bias: 128-query hand-offs
           return !bm ? evo::launch_bwd_nb_bf16(F, dpad(d->D), st)
                      : evo::launch_bwd_pb_bf16(F, dpad(d->D), st);
         })) != cudaSuccess)
      return cuda_fail(e, "bwd_fused");
    if (big) {
      ++nl;
      fa.t0 = 2;
      fa.sigma_only = 1;
      if ((e = traced(st, "bwd_fused_sigma", [&] { return evo::launch_bwd_pb_bf16(F, dpad(d->D), st); })) != cudaSuccess) return cuda_fail(e, "bwd_pb (sigma pass)");
    }
    ++nl;
    // fork: the dbias reduce runs on the side stream while dq_convert runs on the caller's
    SideStream* ss = (dqacc && bm) ? side_stream() : nullptr;
    cudaStream_t rst = st;
    if (ss && cudaEventRecord(ss->fork, st) == cudaSuccess &&
        cudaStreamWaitEvent(ss->s, ss->fork, 0) == cudaSuccess)
      rst = ss->s;
    else
      (void)cudaGetLastError();
    if (bm) {
      evo::ReduceArgs ra{};
      ra.nparts = fa.nchunks; ra.H = d->H; ra.Lq = d->Lq; ra.Lk = d->Lk; ra.nb = 1;
      ra.partial = fa.partial; ra.dbias = dbias;
      ra.s_b = 0; ra.s_h = d->bias_str[1]; ra.s_q = d->bias_str[2]; ra.s_k = d->bias_str[3];
      ra.q_fast = bm == 2;
      if ((e = traced(rst, "dbias_reduce", [&] { return evo::launch_dbias_reduce(ra, rst); })) != cudaSuccess) return cuda_fail(e, "dbias_reduce");
      ++nl;
    }
    if (dqacc) {
      evo::ConvertArgs ca{};
      ca.B = (int)d->B; ca.H = d->H; ca.Lq = d->Lq; ca.D = d->D; ca.scale = d->scale; ca.acc = dqacc;
      ca.nparts = fa.dq_reduce ? 1 : nk; ca.part_stride = (int64_t)d->B * d->H * d->Lq * d->D;
      ca.p_sb = part_str[0]; ca.p_sh = part_str[1]; ca.p_sl = part_str[2];
      ca.dq = (__nv_bfloat16*)dq; ca.q_sb = d->q_str[0]; ca.q_sh = d->q_str[1]; ca.q_sl = d->q_str[2];
      if ((e = traced(st, "dq_convert", [&] { return evo::launch_dq_convert(ca, st); })) != cudaSuccess) return cuda_fail(e, "dq_convert");
      ++nl;
    }
    if (rst != st) {  // join
      if ((e = cudaEventRecord(ss->join, rst)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(st, ss->join, 0)) != cudaSuccess)
        return cuda_fail(e, "side-stream join");
    }
    g_launches = nl;
    return EVO_OK;
  }
  evo::BwdMainLaunch M;
  M.tm_q = tq; M.tm_k = tk; M.tm_v = tv; M.tm_da = tda; M.tm_b = tb;
  evo::BwdMainArgs& ma = M.args;
  memset(&ma, 0, sizeof(ma));
  ma.B = (int)d->B; ma.H = d->H; ma.Lq = d->Lq; ma.Lk = d->Lk; ma.D = d->D;
  ma.scale = d->scale; ma.scale_log2 = d->scale * evo::kLog2e;
  ma.bias_batched = d->bias_kind == EVO_BIAS_PER_BATCH;
  ma.mask = mask; ma.mask_s0 = d->mask_str[0]; ma.mask_s1 = d->mask_str[1];
  ma.lse2 = lse2; ma.Dvec = dvec;
  ma.dk = (__nv_bfloat16*)dk; ma.k_sb = d->k_str[0]; ma.k_sh = d->k_str[1]; ma.k_sl = d->k_str[2];
  ma.dv = (__nv_bfloat16*)dv; ma.v_sb = d->v_str[0]; ma.v_sh = d->v_str[1]; ma.v_sl = d->v_str[2];
  ma.dq = (__nv_bfloat16*)dq; ma.q_sb = d->q_str[0]; ma.q_sh = d->q_str[1]; ma.q_sl = d->q_str[2];
  ma.dq_acc = dqacc;
  if ((e = traced(st, "bwd_main", [&] { return evo::launch_bwd_main_bf16(M, dpad(d->D), bm, st); })) != cudaSuccess) return cuda_fail(e, "bwd_main");
  ++nl;
  if (dqacc) {
    evo::ConvertArgs ca{};
    ca.B = (int)d->B; ca.H = d->H; ca.Lq = d->Lq; ca.D = d->D; ca.scale = d->scale; ca.acc = dqacc;
    ca.nparts = nk;  // bwd_main's per-key-tile parts [nk][B,H,Lq,D], summed in key-tile order
    ca.part_stride = (int64_t)d->B * d->H * d->Lq * d->D;
    ca.p_sb = (int64_t)d->H * d->Lq * d->D; ca.p_sh = (int64_t)d->Lq * d->D; ca.p_sl = d->D;
    ca.dq = (__nv_bfloat16*)dq; ca.q_sb = d->q_str[0]; ca.q_sh = d->q_str[1]; ca.q_sl = d->q_str[2];
    if ((e = traced(st, "dq_convert", [&] { return evo::launch_dq_convert(ca, st); })) != cudaSuccess) return cuda_fail(e, "dq_convert");
    ++nl;
  }
  if (bm) {
    evo::BwdBiasLaunch Bl;
    Bl.tm_q = tq; Bl.tm_k = tk; Bl.tm_v = tv; Bl.tm_da = tda; Bl.tm_b = tb;
    evo::BwdBiasArgs& ba = Bl.args;
    memset(&ba, 0, sizeof(ba));
    ba.B = (int)d->B; ba.H = d->H; ba.Lq = d->Lq; ba.Lk = d->Lk; ba.D = d->D;
    ba.scale_log2 = d->scale * evo::kLog2e;
    ba.bias_batched = d->bias_kind == EVO_BIAS_PER_BATCH;
    ba.nchunks = W.nchunks; ba.chunk = W.chunk;
    ba.mask = mask; ba.mask_s0 = d->mask_str[0]; ba.mask_s1 = d->mask_str[1];
    ba.lse2 = lse2; ba.Dvec = dvec;
    ba.partial = reinterpret_cast<float*>(ws + W.partial);
    if ((e = traced(st, "bwd_bias", [&] { return evo::launch_bwd_bias_bf16(Bl, dpad(d->D), bm, st); })) != cudaSuccess) return cuda_fail(e, "bwd_bias");
    ++nl;
    evo::ReduceArgs ra{};
    const bool pb = d->bias_kind == EVO_BIAS_PER_BATCH;
    ra.nparts = pb ? 1 : W.nchunks; ra.H = d->H; ra.Lq = d->Lq; ra.Lk = d->Lk;
    ra.nb = pb ? d->B : 1;
    ra.partial = ba.partial; ra.dbias = dbias;
    ra.s_b = pb ? d->bias_str[0] : 0; ra.s_h = d->bias_str[1]; ra.s_q = d->bias_str[2]; ra.s_k = d->bias_str[3];
    ra.q_fast = bm == 2;
    if ((e = traced(st, "dbias_reduce", [&] { return evo::launch_dbias_reduce(ra, st); })) != cudaSuccess) return cuda_fail(e, "dbias_reduce");
    ++nl;
  }
  g_launches = nl;
  return EVO_OK;
}

}  // extern "C"
