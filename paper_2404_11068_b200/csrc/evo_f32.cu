// evo_f32.cu — fp32 verification mode (EVO_F32): the same operation entirely in fp32 FFMA with
// accurate expf/logf on the SIMT pipes (tf32 tensor cores cannot meet the 1e-5 bar of the north
// star).  Not a fast path; it exists to lock semantics (mask, gate, bias broadcast/orientation,
// fully-masked rows) at 1e-5 against the fp64 oracle.
#include "evo_kernels.cuh"

namespace evo {

constexpr int kF32Keys = 32;  // keys (or queries) staged in shared memory per step

EVO_DEV float bias_f32(const F32Args& a, int64_t b, int h, int q, int k) {
  if (a.bias_kind == 0) return 0.f;
  const int64_t bb = a.bias_kind == 2 ? b : 0;
  return a.bias[bb * a.b_sb + (int64_t)h * a.b_sh + (int64_t)q * a.b_sq + (int64_t)k * a.b_sk];
}
EVO_DEV bool keep_f32(const F32Args& a, int64_t b, int k) {
  return a.mask == nullptr || a.mask[b * a.mask_s0 + (int64_t)k * a.mask_s1] != 0;
}

// ------------------------------------------------------------------ forward: thread = query row
__global__ void __launch_bounds__(128) fwd_f32_kernel(const F32Args a) {
  __shared__ float sk[kF32Keys][64], sv[kF32Keys][64];
  const int nq = (a.Lq + 127) / 128;
  const int qt = blockIdx.x % nq;
  const int bh = blockIdx.x / nq;
  const int h = bh % a.H;
  const int64_t b = bh / a.H;
  const int q = qt * 128 + threadIdx.x;
  const bool qv = q < a.Lq;
  float qr[64], acc[64];
  for (int d = 0; d < a.D; ++d) {
    qr[d] = qv ? a.q[b * a.q_sb + h * a.q_sh + (int64_t)q * a.q_sl + d] : 0.f;
    acc[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < a.Lk; k0 += kF32Keys) {
    __syncthreads();
    for (int t = threadIdx.x; t < kF32Keys * a.D; t += blockDim.x) {
      const int kk = t / a.D, d = t % a.D, k = k0 + kk;
      sk[kk][d] = k < a.Lk ? a.k[b * a.k_sb + h * a.k_sh + (int64_t)k * a.k_sl + d] : 0.f;
      sv[kk][d] = k < a.Lk ? a.v[b * a.v_sb + h * a.v_sh + (int64_t)k * a.v_sl + d] : 0.f;
    }
    __syncthreads();
    if (!qv) continue;
    for (int kk = 0; kk < kF32Keys && k0 + kk < a.Lk; ++kk) {
      const int k = k0 + kk;
      if (!keep_f32(a, b, k)) continue;
      float s = 0.f;
      for (int d = 0; d < a.D; ++d) s = fmaf(qr[d], sk[kk][d], s);
      s = a.scale * s + bias_f32(a, b, h, q, k);
      const float mn = fmaxf(m, s);
      const float corr = expf(m - mn);  // m = -inf -> 0
      const float p = expf(s - mn);
      l = l * corr + p;
      for (int d = 0; d < a.D; ++d) acc[d] = fmaf(p, sv[kk][d], acc[d] * corr);
      m = mn;
    }
  }
  if (!qv) return;
  const float inv = l > 0.f ? 1.f / l : 0.f;
  for (int d = 0; d < a.D; ++d) {
    float gv = 1.f;
    if (a.g) gv = 1.f / (1.f + expf(-a.g[b * a.g_sb + h * a.g_sh + (int64_t)q * a.g_sl + d]));
    a.o[b * a.o_sb + h * a.o_sh + (int64_t)q * a.o_sl + d] = acc[d] * inv * gv;
  }
  a.lse[(b * a.H + h) * a.Lq + q] = l > 0.f ? m + logf(l) : -INFINITY;
}

cudaError_t launch_fwd_f32(const F32Args& a, cudaStream_t st) {
  const long long grid = (long long)a.B * a.H * ((a.Lq + 127) / 128);
  if (grid == 0) return cudaSuccess;
  fwd_f32_kernel<<<(unsigned)grid, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ backward pieces
// dA rows come from a.dA with strides (a_sb, a_sh, a_sl); Dvec / lse_in are [B*H][Lq_pad].
EVO_DEV float prob_f32(const F32Args& a, int64_t b, int h, int q, int k, float s_raw, float lse) {
  if (lse == -INFINITY || !keep_f32(a, b, k)) return 0.f;
  return expf(a.scale * s_raw + bias_f32(a, b, h, q, k) - lse);
}

// dq: thread = query row
__global__ void __launch_bounds__(128) bwd_dq_f32_kernel(const F32Args a) {
  __shared__ float sk[kF32Keys][64], sv[kF32Keys][64];
  const int nq = (a.Lq + 127) / 128, Lq_pad = nq * 128;
  const int qt = blockIdx.x % nq;
  const int bh = blockIdx.x / nq;
  const int h = bh % a.H;
  const int64_t b = bh / a.H;
  const int q = qt * 128 + threadIdx.x;
  const bool qv = q < a.Lq;
  float qr[64], da[64], dq[64];
  for (int d = 0; d < a.D; ++d) {
    qr[d] = qv ? a.q[b * a.q_sb + h * a.q_sh + (int64_t)q * a.q_sl + d] : 0.f;
    da[d] = qv ? a.dA[b * a.a_sb + h * a.a_sh + (int64_t)q * a.a_sl + d] : 0.f;
    dq[d] = 0.f;
  }
  const float lse = qv ? a.lse_in[(b * a.H + h) * a.Lq + q] : -INFINITY;
  const float Dq = qv ? a.Dvec[(int64_t)bh * Lq_pad + q] : 0.f;
  for (int k0 = 0; k0 < a.Lk; k0 += kF32Keys) {
    __syncthreads();
    for (int t = threadIdx.x; t < kF32Keys * a.D; t += blockDim.x) {
      const int kk = t / a.D, d = t % a.D, k = k0 + kk;
      sk[kk][d] = k < a.Lk ? a.k[b * a.k_sb + h * a.k_sh + (int64_t)k * a.k_sl + d] : 0.f;
      sv[kk][d] = k < a.Lk ? a.v[b * a.v_sb + h * a.v_sh + (int64_t)k * a.v_sl + d] : 0.f;
    }
    __syncthreads();
    if (!qv) continue;
    for (int kk = 0; kk < kF32Keys && k0 + kk < a.Lk; ++kk) {
      const int k = k0 + kk;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < a.D; ++d) {
        s = fmaf(qr[d], sk[kk][d], s);
        dp = fmaf(da[d], sv[kk][d], dp);
      }
      const float p = prob_f32(a, b, h, q, k, s, lse);
      const float ds = p * (dp - Dq);
      for (int d = 0; d < a.D; ++d) dq[d] = fmaf(ds, sk[kk][d], dq[d]);
    }
  }
  if (!qv) return;
  for (int d = 0; d < a.D; ++d) a.dq[b * a.q_sb + h * a.q_sh + (int64_t)q * a.q_sl + d] = a.scale * dq[d];
}

// dk, dv: thread = key row
__global__ void __launch_bounds__(128) bwd_dkdv_f32_kernel(const F32Args a) {
  __shared__ float sq[kF32Keys][64], sa[kF32Keys][64], sl[kF32Keys], sd[kF32Keys];
  const int nk = (a.Lk + 127) / 128, Lq_pad = ((a.Lq + 127) / 128) * 128;
  const int kt = blockIdx.x % nk;
  const int bh = blockIdx.x / nk;
  const int h = bh % a.H;
  const int64_t b = bh / a.H;
  const int k = kt * 128 + threadIdx.x;
  const bool kv = k < a.Lk;
  float kr[64], vr[64], dk[64], dv[64];
  for (int d = 0; d < a.D; ++d) {
    kr[d] = kv ? a.k[b * a.k_sb + h * a.k_sh + (int64_t)k * a.k_sl + d] : 0.f;
    vr[d] = kv ? a.v[b * a.v_sb + h * a.v_sh + (int64_t)k * a.v_sl + d] : 0.f;
    dk[d] = 0.f;
    dv[d] = 0.f;
  }
  for (int q0 = 0; q0 < a.Lq; q0 += kF32Keys) {
    __syncthreads();
    for (int t = threadIdx.x; t < kF32Keys * a.D; t += blockDim.x) {
      const int qq = t / a.D, d = t % a.D, q = q0 + qq;
      sq[qq][d] = q < a.Lq ? a.q[b * a.q_sb + h * a.q_sh + (int64_t)q * a.q_sl + d] : 0.f;
      sa[qq][d] = q < a.Lq ? a.dA[b * a.a_sb + h * a.a_sh + (int64_t)q * a.a_sl + d] : 0.f;
    }
    for (int t = threadIdx.x; t < kF32Keys; t += blockDim.x) {
      const int q = q0 + t;
      sl[t] = q < a.Lq ? a.lse_in[(b * a.H + h) * a.Lq + q] : -INFINITY;
      sd[t] = q < a.Lq ? a.Dvec[(int64_t)bh * Lq_pad + q] : 0.f;
    }
    __syncthreads();
    if (!kv) continue;
    for (int qq = 0; qq < kF32Keys && q0 + qq < a.Lq; ++qq) {
      const int q = q0 + qq;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < a.D; ++d) {
        s = fmaf(sq[qq][d], kr[d], s);
        dp = fmaf(sa[qq][d], vr[d], dp);
      }
      const float p = prob_f32(a, b, h, q, k, s, sl[qq]);
      const float ds = p * (dp - sd[qq]);
      for (int d = 0; d < a.D; ++d) {
        dv[d] = fmaf(p, sa[qq][d], dv[d]);
        dk[d] = fmaf(ds, sq[qq][d], dk[d]);
      }
    }
  }
  if (!kv) return;
  for (int d = 0; d < a.D; ++d) {
    a.dk[b * a.k_sb + h * a.k_sh + (int64_t)k * a.k_sl + d] = a.scale * dk[d];
    a.dv[b * a.v_sb + h * a.v_sh + (int64_t)k * a.v_sl + d] = dv[d];
  }
}

// dbias: thread = (q, k) of one head (and one b for the per-batch kind); Σ over b in order
__global__ void __launch_bounds__(256) bwd_dbias_f32_kernel(const F32Args a) {
  const int Lq_pad = ((a.Lq + 127) / 128) * 128;
  const int64_t nb = a.bias_kind == 2 ? a.B : 1;
  const int64_t n = nb * a.H * (int64_t)a.Lq * a.Lk;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = idx;
    const int k = (int)(t % a.Lk); t /= a.Lk;
    const int q = (int)(t % a.Lq); t /= a.Lq;
    const int h = (int)(t % a.H);
    const int64_t bsel = t / a.H;
    const int64_t b_lo = a.bias_kind == 2 ? bsel : 0, b_hi = a.bias_kind == 2 ? bsel + 1 : a.B;
    float sum = 0.f;
    for (int64_t b = b_lo; b < b_hi; ++b) {
      const float lse = a.lse_in[(b * a.H + h) * a.Lq + q];
      if (lse == -INFINITY || !keep_f32(a, b, k)) continue;
      const float* qp = a.q + b * a.q_sb + h * a.q_sh + (int64_t)q * a.q_sl;
      const float* kp = a.k + b * a.k_sb + h * a.k_sh + (int64_t)k * a.k_sl;
      const float* vp = a.v + b * a.v_sb + h * a.v_sh + (int64_t)k * a.v_sl;
      const float* ap = a.dA + b * a.a_sb + h * a.a_sh + (int64_t)q * a.a_sl;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < a.D; ++d) {
        s = fmaf(qp[d], kp[d], s);
        dp = fmaf(ap[d], vp[d], dp);
      }
      const float p = expf(a.scale * s + bias_f32(a, b, h, q, k) - lse);
      sum += p * (dp - a.Dvec[(b * a.H + h) * Lq_pad + q]);
    }
    a.dbias[bsel * (a.bias_kind == 2 ? a.b_sb : 0) + (int64_t)h * a.b_sh + (int64_t)q * a.b_sq +
            (int64_t)k * a.b_sk] = sum;
  }
}

cudaError_t launch_bwd_f32(const F32Args& a, cudaStream_t st, int* nlaunch) {
  const long long gq = (long long)a.B * a.H * ((a.Lq + 127) / 128);
  const long long gk = (long long)a.B * a.H * ((a.Lk + 127) / 128);
  if (gq > 0) { bwd_dq_f32_kernel<<<(unsigned)gq, 128, 0, st>>>(a); ++*nlaunch; }
  if (gk > 0) { bwd_dkdv_f32_kernel<<<(unsigned)gk, 128, 0, st>>>(a); ++*nlaunch; }
  if (a.bias_kind != 0 && a.dbias) {
    const int64_t nb = a.bias_kind == 2 ? a.B : 1;
    const int64_t n = nb * a.H * (int64_t)a.Lq * a.Lk;
    if (n > 0) {
      const int64_t blocks = (n + 255) / 256;
      bwd_dbias_f32_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(a);
      ++*nlaunch;
    }
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Lk == 0: every row empty
__global__ void fill_empty_kernel(float* lse, int64_t nrows, void* o, int f32, int B, int H,
                                  int Lq, int D, int64_t o_sb, int64_t o_sh, int64_t o_sl) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    lse[r] = -INFINITY;
    const int q = (int)(r % Lq);
    const int64_t bh = r / Lq;
    const int h = (int)(bh % H);
    const int64_t b = bh / H;
    const int64_t base = b * o_sb + h * o_sh + (int64_t)q * o_sl;
    for (int d = 0; d < D; ++d) {
      if (f32) reinterpret_cast<float*>(o)[base + d] = 0.f;
      else reinterpret_cast<__nv_bfloat16*>(o)[base + d] = __float2bfloat16(0.f);
    }
  }
}

cudaError_t launch_fill_empty(float* lse, int64_t nrows, void* o, int dtype, int B, int H,
                              int Lq, int D, int64_t o_sb, int64_t o_sh, int64_t o_sl,
                              cudaStream_t st) {
  if (nrows == 0) return cudaSuccess;
  const int64_t blocks = (nrows + 255) / 256;
  fill_empty_kernel<<<(unsigned)(blocks < 1184 ? blocks : 1184), 256, 0, st>>>(
      lse, nrows, o, dtype == 1, B, H, Lq, D, o_sb, o_sh, o_sl);
  return cudaGetLastError();
}

}  // namespace evo
