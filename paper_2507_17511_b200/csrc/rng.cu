// Device draw of the reference's low-rank start block, bit-identical to numpy:
//   Q0 = float32(Generator(PCG64(SeedSequence(entropy, spawn_key))).standard_normal((rows, cols)))
// (compressors.py:407 -> linalg.py:67-74, rng from linalg.py:25-27 with the keys of
// pipeline.py:190 / mesh.py:193).  Drawing it here instead of on the host takes
// the ~0.26 ms numpy draw off the step and makes the low-rank step capturable in
// a CUDA graph: the key's step word lives in device memory and is advanced by
// the kernel, so every replay draws the next step's block.
//
// Algorithms (restated and pinned to numpy in oracle/np_random.py):
//   SeedSequence  hash-mix of the assembled entropy words into a 4-word pool,
//                 generate_state(4, uint64) -> PCG64 srandom(initstate, initseq)
//   PCG64         128-bit LCG, XSL-RR 64-bit output, O(log n) jump-ahead
//   normal        numpy's 256-level ziggurat (random_standard_normal): a draw is
//                 one u64 on the fast path (~99% of draws); the wedge / tail paths
//                 consume further u64s, so the stream positions of the draws are
//                 data dependent.
// Parallel form (two launches):
//   k_gauss_gen   CTA c generates stream positions [c P, (c + 1) P) by jump-ahead
//                 (16 per thread) and lists the positions that fail the fast test;
//                 the last CTA to finish (ticket) evaluates every listed position AS
//                 IF a draw started there (value, u64s consumed), decides which of
//                 them really start a draw (a listed position is skipped when a real
//                 slow draw before it consumed it: short ranges, resolved in a few
//                 parallel rounds) and, by a scan, the output index of each real slow
//                 draw and the position shift of the draws after it
//   k_gauss_out   every output index maps to its stream position (fast draw) or to
//                 an evaluated slow draw, by a binary search over the shifts
// Floating point follows numpy's C expression order with no contraction; exp /
// log1p are CUDA's (<= 1 ulp from glibc), which can only matter when a wedge / tail
// acceptance test or the f32 rounding of a tail value lands within an ulp.
#include "cc_common.cuh"
#include "cc_internal.h"
#include "ziggurat_tables.h"

namespace cc {
namespace rng {

using u128 = unsigned __int128;
constexpr int kThreads = 1024;
constexpr int kMaxWords = 16;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}
__device__ __forceinline__ uint64_t pcg_out(u128 s) {  // XSL-RR
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// SeedSequence(entropy, spawn_key) -> PCG64 (state, inc)
__device__ void seed_pcg(const uint32_t *w, int nw, u128 &state, u128 &inc) {
  constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? w[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(w[s]));
  uint32_t out[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    out[i] = v;
  }
  uint64_t v64[4];
  for (int i = 0; i < 4; ++i) v64[i] = (uint64_t)out[2 * i] | ((uint64_t)out[2 * i + 1] << 32);
  const u128 initstate = ((u128)v64[0] << 64) | v64[1];
  const u128 initseq = ((u128)v64[2] << 64) | v64[3];
  inc = (initseq << 1) | 1;
  u128 s = inc;  // state = 0; step
  s += initstate;
  state = s * pcg_mult() + inc;  // step
}

__device__ __forceinline__ double next_double(uint64_t u) { return __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0); }

struct Shared {
  u128 state0, inc;
  uint32_t nslow, nev;
  uint32_t wsum[kThreads / 32];
};

// one draw of random_standard_normal starting at stream position p (raw[p] = the
// (p+1)-th output); returns the value and sets *next to the first unused position
// the ziggurat tables staged in shared memory (random per-lane indices: a gather from
// shared memory instead of a serialised constant-cache access)
struct Zig {
  const uint64_t *ki;
  const double *wi, *fi;
};

__device__ __forceinline__ void stage_tables(uint64_t *ki, double *wi, double *fi) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    ki[i] = zig::kKi[i];
    wi[i] = zig::kWi[i];
    fi[i] = zig::kFi[i];
  }
}

__device__ double draw_at(const uint64_t *raw, int64_t npos, const Shared &sh, const Zig &zt, int64_t p,
                          int64_t *next) {
  auto raw_at = [&](int64_t q) -> uint64_t {
    return q < npos ? __ldcg(raw + q) : pcg_out(pcg_advance(sh.state0, sh.inc, (uint64_t)q + 1));
  };
  for (;;) {
    uint64_t r = raw_at(p++);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const uint64_t sign = r & 1, rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, zt.wi[idx]);
    if (sign) x = -x;
    if (rabs < zt.ki[idx]) {
      *next = p;
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-zig::kNorInvR, log1p(-next_double(raw_at(p++))));
        const double yy = -log1p(-next_double(raw_at(p++)));
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          *next = p;
          return ((rabs >> 8) & 1) ? -__dadd_rn(zig::kNorR, xx) : __dadd_rn(zig::kNorR, xx);
        }
      }
    } else {
      const double f = __dadd_rn(__dmul_rn(__dsub_rn(zt.fi[idx - 1], zt.fi[idx]), next_double(raw_at(p++))),
                                 zt.fi[idx]);
      if (f < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
        *next = p;
        return x;
      }
    }
  }
}

struct Work {
  uint64_t *raw;      // [npos]
  uint32_t *cand;     // [nblk][kGenPos] positions failing the fast test (per-CTA segment, ascending)
  uint32_t *ncand;    // [nblk]
  uint32_t *ev_o;     // [kMaxEv] output index of each real slow draw (ascending)
  uint32_t *ev_sh;    // [kMaxEv] position shift (pos - out) of the draws after it
  double *ev_v;       // [kMaxEv]
  uint32_t *ctl;      // [1] event count (workspace)
  uint32_t *ticket;   // last-CTA ticket: a library-owned zeroed word (left zero by every launch)
  uint32_t *sslow;    // [npos] sequential-walk fallback: all candidates in order
  uint32_t *scons;    // [npos]
  double *sval;       // [npos]
};

constexpr int kGenThreads = 256, kGenPer = 16, kGenPos = kGenThreads * kGenPer;  // positions per CTA
constexpr int kMaxCand = 2048;  // slow candidates resolved in shared memory (~0.7% of positions)
constexpr int kMaxEv = kMaxCand;
constexpr int kOutThreads = 256;

__device__ __forceinline__ bool slow_pos(uint64_t r, const uint64_t *ki) {
  return ((r >> 9) & 0x000fffffffffffffull) >= ki[r & 0xff];
}

__device__ unsigned long long *g_gauss_stamps = nullptr;  // profiling: [16] %globaltimer stamps

__device__ __forceinline__ void gstamp(int i) {
  if (g_gauss_stamps && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_gauss_stamps[i] = t;
  }
}

__global__ void __launch_bounds__(kGenThreads) k_gauss_gen(const uint32_t *__restrict__ key, int nw, int64_t M,
                                                            int64_t npos, Work w) {
  __shared__ Shared sh;
  __shared__ uint32_t wcnt[kGenThreads / 32], s_last;
  __shared__ uint32_t c_pos[kMaxCand];
  __shared__ uint8_t c_cons[kMaxCand], c_real[kMaxCand];
  __shared__ double c_val[kMaxCand];
  __shared__ uint64_t tki[256];
  __shared__ double twi[256], tfi[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  stage_tables(tki, twi, tfi);
  const Zig zt{tki, twi, tfi};
  if (blockIdx.x == 0) gstamp(0);
  if (tid == 0) {
    uint32_t kw[kMaxWords];
    for (int i = 0; i < nw; ++i) kw[i] = key[i];
    seed_pcg(kw, nw, sh.state0, sh.inc);
  }
  __syncthreads();
  if (blockIdx.x == 0) gstamp(1);
  // ---- generate this thread's kGenPer positions ----
  const int64_t p0 = (int64_t)blockIdx.x * kGenPos + (int64_t)tid * kGenPer;
  uint32_t slowmask = 0;
  {
    u128 st = pcg_advance(sh.state0, sh.inc, (uint64_t)p0);
    const u128 m = pcg_mult(), inc = sh.inc;
#pragma unroll
    for (int k = 0; k < kGenPer; ++k) {
      st = st * m + inc;
      if (p0 + k < npos) {
        const uint64_t r = pcg_out(st);
        w.raw[p0 + k] = r;
        slowmask |= (uint32_t)slow_pos(r, tki) << k;
      }
    }
  }
  if (blockIdx.x == 0) gstamp(2);
  // ---- this CTA's candidate list (ascending), per-CTA segment ----
  const uint32_t nl = __popc(slowmask);
  uint32_t incl = nl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wcnt[warp] = incl;
  __syncthreads();
  uint32_t off = incl - nl;
  for (int i = 0; i < warp; ++i) off += wcnt[i];
  uint32_t *seg = w.cand + (size_t)blockIdx.x * kGenPos;
  for (uint32_t mm = slowmask; mm; mm &= mm - 1) seg[off++] = (uint32_t)(p0 + __ffs(mm) - 1);
  if (tid == kGenThreads - 1) w.ncand[blockIdx.x] = off;
  // ---- the last CTA resolves the slow draws ----
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(w.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  gstamp(3);
  // gather every CTA's candidates in position order
  __shared__ uint32_t s_nc[1024];
  for (unsigned b = tid; b < gridDim.x && b < 1024; b += kGenThreads) s_nc[b] = __ldcg(w.ncand + b);
  __syncthreads();
  uint32_t total = 0;
  for (unsigned b = 0; b < gridDim.x; ++b) {
    const uint32_t nb = b < 1024 ? s_nc[b] : __ldcg(w.ncand + b);
    for (uint32_t i = tid; i < nb; i += kGenThreads)
      if (total + i < (uint32_t)kMaxCand) c_pos[total + i] = __ldcg(w.cand + (size_t)b * kGenPos + i);
    total += nb;
  }
  __syncthreads();
  if (total > (uint32_t)kMaxCand) {  // never in practice (~1% of positions are slow): sequential walk
    if (tid == 0) {
      uint32_t n = 0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const uint32_t nb = __ldcg(w.ncand + b);
        for (uint32_t i = 0; i < nb; ++i) w.sslow[n++] = __ldcg(w.cand + (size_t)b * kGenPos + i);
      }
      int64_t pos = 0, j = 0;
      uint32_t nev = 0;
      for (uint32_t i = 0; i < n && j < M; ++i) {
        const int64_t p = w.sslow[i];
        if (p < pos) continue;
        const int64_t run = p - pos;
        if (j + run >= M) break;
        j += run;
        int64_t nx;
        const double v = draw_at(w.raw, npos, sh, zt, p, &nx);
        pos = nx;
        if (nev < (uint32_t)kMaxEv) {
          w.ev_o[nev] = (uint32_t)j;
          w.ev_v[nev] = v;
          w.ev_sh[nev] = (uint32_t)(pos - (j + 1));
        }
        ++nev;
        ++j;
      }
      w.ctl[1] = nev;
      *w.ticket = 0u;
    }
    return;
  }
  gstamp(4);
  // evaluate every candidate as a draw start
  for (uint32_t i = tid; i < total; i += kGenThreads) {
    int64_t nx;
    c_val[i] = draw_at(w.raw, npos, sh, zt, c_pos[i], &nx);
    c_cons[i] = (uint8_t)min64(nx - (int64_t)c_pos[i], 255);  // a draw never takes 255 u64s
    c_real[i] = 1u;
  }
  __syncthreads();
  gstamp(5);
  // real starts: a candidate is skipped iff a REAL candidate before it consumed it.
  // Consumed ranges are a few positions long, so only the nearest preceding
  // candidates can cover one; iterate to the fixed point (a couple of rounds).
  __shared__ int changed;
  for (int round = 0; round < 64; ++round) {
    if (tid == 0) changed = 0;
    __syncthreads();
    uint32_t nr[16];
    int nk = 0;
    for (uint32_t k = tid; k < total; k += kGenThreads) {
      uint32_t real = 1u;
      for (int i = (int)k - 1; i >= 0; --i) {
        if ((int64_t)c_pos[i] + 64 < (int64_t)c_pos[k]) break;  // no draw consumes 64 u64s
        if (c_real[i] && c_pos[i] + c_cons[i] > c_pos[k]) {
          real = 0u;
          break;
        }
      }
      if (nk < 16) nr[nk] = real;
      ++nk;
    }
    __syncthreads();
    nk = 0;
    for (uint32_t k = tid; k < total; k += kGenThreads) {
      const uint32_t real = nk < 16 ? nr[nk] : 1u;
      ++nk;
      if (real != c_real[k]) {
        c_real[k] = real;
        changed = 1;
      }
    }
    __syncthreads();
    const int ch = changed;
    __syncthreads();  // every thread has read the flag before thread 0 clears it for the next round
    if (!ch) break;
  }
  // output index of real candidate k: p_k minus the extra positions consumed by the
  // real slow draws before it; shift after it = p_k + cons_k - (out_k + 1)
  gstamp(6);
  // block scan over the candidates (thread t: candidates [t K, t K + K)): events
  // before each real one (event slot) and extra positions consumed before it
  {
    constexpr int K = kMaxCand / kGenThreads;
    uint32_t ne = 0, ex = 0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const uint32_t k = tid * K + u;
      if (k < total && c_real[k]) {
        ++ne;
        ex += c_cons[k] - 1u;
      }
    }
    // pack (events, extra) into one 64-bit scan value
    unsigned long long v = ((unsigned long long)ne << 40) | ex, incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __shared__ unsigned long long wsum64[kGenThreads / 32];
    if (lane == 31) wsum64[warp] = incl;
    __syncthreads();
    unsigned long long before = incl - v;
    for (int i = 0; i < warp; ++i) before += wsum64[i];
    uint32_t slot = (uint32_t)(before >> 40), extra = (uint32_t)(before & ((1ull << 40) - 1));
    __shared__ uint32_t s_nev;
    if (tid == 0) s_nev = 0xffffffffu;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const uint32_t k = tid * K + u;
      if (k < total && c_real[k]) {
        const int64_t o = (int64_t)c_pos[k] - extra;  // output index of this slow draw
        extra += c_cons[k] - 1u;
        if (o < M) {
          w.ev_o[slot] = (uint32_t)o;
          w.ev_v[slot] = c_val[k];
          w.ev_sh[slot] = extra;  // shift (position - output) of the draws after it
        } else {
          atomicMin(&s_nev, slot);  // the first real slow draw at or past M ends the list
        }
        ++slot;
      }
    }
    __syncthreads();
    if (tid == kGenThreads - 1) {
      w.ctl[1] = min(s_nev, slot);
      *w.ticket = 0u;  // ticket ready for the next launch
    }
  }
  __syncthreads();
  gstamp(7);
}

__global__ void __launch_bounds__(kOutThreads) k_gauss_out(uint32_t *key, int nw, int step_word, int64_t M,
                                                            int64_t npos, Work w, float *__restrict__ out) {
  __shared__ Shared sh;
  __shared__ uint32_t s_o[kMaxEv], s_sh[kMaxEv];
  __shared__ uint64_t tki[256];
  __shared__ double twi[256], tfi[256];
  const int tid = threadIdx.x;
  stage_tables(tki, twi, tfi);
  const Zig zt{tki, twi, tfi};
  const uint32_t nev = min(__ldcg(w.ctl + 1), (uint32_t)kMaxEv);
  for (uint32_t i = tid; i < nev; i += kOutThreads) {
    s_o[i] = __ldcg(w.ev_o + i);
    s_sh[i] = __ldcg(w.ev_sh + i);
  }
  if (tid == 0) {
    uint32_t kw[kMaxWords];
    for (int i = 0; i < nw; ++i) kw[i] = key[i];
    seed_pcg(kw, nw, sh.state0, sh.inc);  // only for draws past the generated positions
  }
  __syncthreads();
  if (blockIdx.x == 0) gstamp(8);
  const int64_t j0 = (int64_t)blockIdx.x * kOutThreads * 4 + tid;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t j = j0 + u * kOutThreads;
    if (j >= M) break;
    int lo = 0, hi = (int)nev;  // events [0, lo) have ev_o <= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)s_o[mid] <= j) lo = mid + 1;
      else hi = mid;
    }
    double v;
    if (lo > 0 && (int64_t)s_o[lo - 1] == j) {
      v = __ldcg(w.ev_v + lo - 1);
    } else {
      const int64_t p = j + (lo > 0 ? (int64_t)s_sh[lo - 1] : 0);
      int64_t nx;
      v = draw_at(w.raw, npos, sh, zt, p, &nx);  // a fast draw (or past the generated positions)
    }
    out[j] = (float)v;
  }
  if (blockIdx.x == 0 && tid == 0 && step_word >= 0) key[step_word] += 1u;  // the next step's key
  if (blockIdx.x == 0) {
    __syncthreads();
    gstamp(9);
  }
}

void set_gauss_stamps(void *buf) {
  unsigned long long *p = reinterpret_cast<unsigned long long *>(buf);
  cudaMemcpyToSymbol(g_gauss_stamps, &p, sizeof(p));
}

static int64_t npos_for(int64_t M) { return M + M / 8 + 1024; }

static Work carve(void *ws, int64_t npos, size_t *bytes) {
  Work w{};
  uint8_t *b = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t sz) {
    uint8_t *q = b ? b + off : nullptr;
    off = align_up(off + sz, 256);
    return q;
  };
  const int64_t nblk = cdiv(npos, kGenPos);
  w.raw = reinterpret_cast<uint64_t *>(take(8 * npos));
  w.cand = reinterpret_cast<uint32_t *>(take(4 * (size_t)nblk * kGenPos));
  w.ncand = reinterpret_cast<uint32_t *>(take(4 * nblk));
  w.ev_o = reinterpret_cast<uint32_t *>(take(4 * kMaxEv));
  w.ev_sh = reinterpret_cast<uint32_t *>(take(4 * kMaxEv));
  w.ev_v = reinterpret_cast<double *>(take(8 * kMaxEv));
  w.ctl = reinterpret_cast<uint32_t *>(take(256));
  w.sslow = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.scons = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.sval = reinterpret_cast<double *>(take(8 * npos));
  if (bytes) *bytes = off;
  return w;
}

}  // namespace rng

uint8_t *stream_zero_slab(cudaStream_t st, size_t bytes);
constexpr size_t kGaussTicketOff = 44 * 1024;  // word in the per-stream zeroed slab (top-k: < 34 KB, low-rank: 40 KB)

int64_t gaussian_workspace_bytes(int64_t rows, int64_t cols) {
  size_t b = 0;
  rng::carve(nullptr, rng::npos_for(rows * cols), &b);
  return (int64_t)b;
}

int gaussian_keyed(int64_t rows, int64_t cols, uint32_t *key, int nwords, int step_word, float *out, void *ws,
                   int64_t ws_bytes, cudaStream_t st) {
  const int64_t M = rows * cols;
  if (rows < 1 || cols < 1 || M >= ((int64_t)1 << 31)) {
    set_error("gaussian: bad shape");
    return CC_ERR_SHAPE;
  }
  if (nwords < 1 || nwords > rng::kMaxWords || step_word >= nwords || !key || !out) {
    set_error("gaussian: bad key");
    return CC_ERR_ARG;
  }
  const int64_t npos = rng::npos_for(M);
  size_t need = 0;
  rng::carve(nullptr, npos, &need);
  if ((int64_t)need > ws_bytes) {
    set_error("gaussian workspace too small");
    return CC_ERR_ARG;
  }
  // the last-CTA ticket lives in the stream's zeroed slab (a caller workspace word
  // would carry whatever the allocator's previous user left there)
  uint8_t *slab = stream_zero_slab(st, kGaussTicketOff + 128);
  if (!slab) {
    set_error("gaussian: no control slab (first use inside a capture)");
    return CC_ERR_UNSUPPORTED;
  }
  rng::Work w = rng::carve(ws, npos, nullptr);
  w.ticket = reinterpret_cast<uint32_t *>(slab + kGaussTicketOff);
  const unsigned nblk = (unsigned)cdiv(npos, rng::kGenPos);
  rng::k_gauss_gen<<<nblk, rng::kGenThreads, 0, st>>>(key, nwords, M, npos, w);
  rng::k_gauss_out<<<(unsigned)cdiv(M, 4 * rng::kOutThreads), rng::kOutThreads, 0, st>>>(key, nwords, step_word, M,
                                                                                          npos, w, out);
  count_launch(2);
  return cuda_status("gaussian_keyed");
}

}  // namespace cc
