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
// Parallel form (one CTA): every thread jumps to its slice of stream positions and
// generates them; positions that fail the fast test are evaluated in parallel AS
// IF a draw started there (value, u64s consumed); one thread then walks the short
// list of such positions in order to find which really start a draw and how far
// each shifts the draws after it; finally every output index maps to its position
// (fast draw) or to an evaluated slow draw by a binary search over the shifts.
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
constexpr int kSmemEvents = 4096;  // slow draws searched in shared memory (~1% of the draws)

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
__device__ double draw_at(const uint64_t *raw, int64_t npos, const Shared &sh, int64_t p, int64_t *next) {
  auto raw_at = [&](int64_t q) -> uint64_t {
    return q < npos ? __ldcg(raw + q) : pcg_out(pcg_advance(sh.state0, sh.inc, (uint64_t)q + 1));
  };
  for (;;) {
    uint64_t r = raw_at(p++);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const uint64_t sign = r & 1, rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, zig::kWi[idx]);
    if (sign) x = -x;
    if (rabs < zig::kKi[idx]) {
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
      const double f = __dadd_rn(__dmul_rn(__dsub_rn(zig::kFi[idx - 1], zig::kFi[idx]), next_double(raw_at(p++))),
                                 zig::kFi[idx]);
      if (f < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
        *next = p;
        return x;
      }
    }
  }
}

struct Work {
  uint64_t *raw;    // [npos]
  uint32_t *slow;   // [npos] positions failing the fast test, ascending
  double *sval;     // [npos] value of a draw starting there
  uint32_t *scons;  // [npos] u64s it consumes
  uint32_t *ev_o;   // [npos] output index of each real slow draw
  uint32_t *ev_sh;  // [npos] position shift (pos - out) of the draws after it
  double *ev_v;     // [npos]
};

__global__ void __launch_bounds__(kThreads, 1) k_gauss(uint32_t *key, int nw, int step_word, int64_t M, int64_t npos,
                                                       Work w, float *__restrict__ out) {
  __shared__ Shared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    uint32_t kw[kMaxWords];
    for (int i = 0; i < nw; ++i) kw[i] = key[i];
    seed_pcg(kw, nw, sh.state0, sh.inc);
  }
  __syncthreads();
  // 1. raw stream: thread t generates positions [t cpt, (t + 1) cpt)
  const int64_t cpt = (npos + kThreads - 1) / kThreads;
  const int64_t p0 = min64(npos, (int64_t)tid * cpt), p1 = min64(npos, p0 + cpt);
  uint32_t nslow = 0;
  {
    u128 s = pcg_advance(sh.state0, sh.inc, (uint64_t)p0);
    const u128 m = pcg_mult(), inc = sh.inc;
    for (int64_t p = p0; p < p1; ++p) {
      s = s * m + inc;
      const uint64_t r = pcg_out(s);
      w.raw[p] = r;
      const int idx = (int)(r & 0xff);
      nslow += ((r >> 9) & 0x000fffffffffffffull) >= zig::kKi[idx];
    }
  }
  // 2. ordered list of slow positions (block exclusive scan of the per-thread counts)
  uint32_t incl = nslow;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh.wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = sh.wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    sh.wsum[lane] = v;
    if (lane == 31) sh.nslow = v;
  }
  __syncthreads();
  {
    uint32_t o = (warp ? sh.wsum[warp - 1] : 0u) + incl - nslow;
    for (int64_t p = p0; p < p1; ++p) {
      const uint64_t r = w.raw[p];
      if (((r >> 9) & 0x000fffffffffffffull) >= zig::kKi[r & 0xff]) w.slow[o++] = (uint32_t)p;
    }
  }
  __syncthreads();
  const uint32_t ns = sh.nslow;
  // 3. every slow position evaluated as a draw start
  for (uint32_t i = tid; i < ns; i += kThreads) {
    int64_t nx;
    w.sval[i] = draw_at(w.raw, npos, sh, w.slow[i], &nx);
    w.scons[i] = (uint32_t)(nx - w.slow[i]);
  }
  __syncthreads();
  // 4. walk: which slow positions start a draw, and the position shift after each
  if (tid == 0) {
    int64_t pos = 0, j = 0;
    uint32_t nev = 0;
    for (uint32_t i = 0; i < ns && j < M; ++i) {
      const int64_t p = w.slow[i];
      if (p < pos) continue;  // consumed inside an earlier slow draw
      const int64_t run = p - pos;
      if (j + run >= M) break;  // the remaining draws are all fast
      j += run;
      pos = p + w.scons[i];
      w.ev_o[nev] = (uint32_t)j;
      w.ev_v[nev] = w.sval[i];
      w.ev_sh[nev] = (uint32_t)(pos - (j + 1));
      ++nev;
      ++j;
    }
    sh.nev = nev;
  }
  __syncthreads();
  const uint32_t nev = sh.nev;
  // the event indices and shifts in shared memory for the searches (global beyond)
  __shared__ uint32_t s_o[kSmemEvents], s_sh[kSmemEvents];
  const bool in_smem = nev <= (uint32_t)kSmemEvents;
  if (in_smem) {
    for (uint32_t i = tid; i < nev; i += kThreads) {
      s_o[i] = __ldcg(w.ev_o + i);
      s_sh[i] = __ldcg(w.ev_sh + i);
    }
  }
  __syncthreads();
  const uint32_t *eo = in_smem ? s_o : w.ev_o;
  const uint32_t *esh = in_smem ? s_sh : w.ev_sh;
  // 5. outputs: fast draw at position j + shift, or an evaluated slow draw
  for (int64_t j = tid; j < M; j += kThreads) {
    // last event with ev_o <= j
    int lo = 0, hi = (int)nev;  // invariant: events [0, lo) have ev_o <= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)eo[mid] <= j) lo = mid + 1;
      else hi = mid;
    }
    double v;
    if (lo > 0 && (int64_t)eo[lo - 1] == j) {
      v = __ldcg(w.ev_v + lo - 1);
    } else {
      const int64_t p = j + (lo > 0 ? (int64_t)esh[lo - 1] : 0);
      int64_t nx;
      v = draw_at(w.raw, npos, sh, p, &nx);  // fast path (or past the generated positions)
    }
    out[j] = (float)v;
  }
  if (tid == 0 && step_word >= 0) key[step_word] += 1u;  // the next step's key (graph replays)
}

// generated stream positions: ~1% of draws take the slow paths and consume a few
// extra u64s, so M / 8 + 1024 spare positions are never exhausted in practice; a
// draw that still reaches past them is evaluated from jump-ahead states (correct
// as long as no slow draw starts beyond the generated positions)
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
  w.raw = reinterpret_cast<uint64_t *>(take(8 * npos));
  w.slow = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.sval = reinterpret_cast<double *>(take(8 * npos));
  w.scons = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.ev_o = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.ev_sh = reinterpret_cast<uint32_t *>(take(4 * npos));
  w.ev_v = reinterpret_cast<double *>(take(8 * npos));
  if (bytes) *bytes = off;
  return w;
}

}  // namespace rng

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
  rng::k_gauss<<<1, rng::kThreads, 0, st>>>(key, nwords, step_word, M, npos, rng::carve(ws, npos, nullptr), out);
  count_launch();
  return cuda_status("gaussian_keyed");
}

}  // namespace cc
