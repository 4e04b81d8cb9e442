/* One patch-parallel layer step from plain C, no Python: the C-ABI exchange
 * (cc_allgather_*) over an NCCL communicator built from a unique id, checked
 * against the step's own building blocks (cc_warmup_step / cc_encode_step /
 * cc_decode_step on separately allocated state) — bodies, sender base and the
 * loopback receiver's reconstruction must be bit-identical every step.
 *
 *   gcc -O2 exchange_demo.c -I../../include -I/usr/local/cuda/include \
 *       -L<lib dir> -lcompactcomm_b200 -L/usr/local/cuda/lib64 -lcudart -o demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "compactcomm.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != 0) {                                                               \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,      \
              cc_last_error());                                                   \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static uint16_t to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fff + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}

static int same(const void *a, const void *b, size_t bytes) {
  void *ha = malloc(bytes), *hb = malloc(bytes);
  cudaMemcpy(ha, a, bytes, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, b, bytes, cudaMemcpyDeviceToHost);
  int eq = memcmp(ha, hb, bytes) == 0;
  free(ha);
  free(hb);
  return eq;
}

int main(void) {
  const int64_t rows = 256, cols = 3072, n = rows * cols;
  const int steps = 5;
  cudaSetDevice(0);
  cudaStream_t st;
  cudaStreamCreate(&st);

  uint8_t id[128];
  cc_comm *comm = NULL;
  CHECK(cc_comm_get_unique_id(id));
  CHECK(cc_comm_init_rank(id, 1, 0, &comm));
  if (cc_comm_size(comm) != 1 || cc_comm_rank(comm) != 0) return 2;

  cc_codec_spec spec = {CC_QUANT2, CC_SCALE_RANK1, 0.0, 0, 0};
  cc_allgather_layer *layer = NULL;
  CHECK(cc_allgather_create(comm, &spec, CC_WITH_FEEDBACK, rows, cols, 1, CC_BF16, &layer));

  /* the same channel by hand: sender state + receiver base */
  float *base, *fb, *rbase;
  uint8_t *body, *ws;
  double *rec;
  int64_t body_max = 2 * n, wsb = cc_workspace_bytes(CC_QUANT2, rows, cols, 0);
  cudaMalloc((void **)&base, 4 * n);
  cudaMalloc((void **)&fb, 4 * n);
  cudaMalloc((void **)&rbase, 4 * n);
  cudaMalloc((void **)&body, body_max);
  cudaMalloc((void **)&ws, wsb);
  cudaMalloc((void **)&rec, 16);
  cudaMemset(base, 0, 4 * n);
  cudaMemset(fb, 0, 4 * n);

  uint16_t *hx = malloc(2 * n);
  uint16_t *dx;
  cudaMalloc((void **)&dx, 2 * n);
  uint32_t seed = 12345u;
  float *cur = calloc(n, sizeof(float));
  for (int t = 1; t <= steps; ++t) {
    for (int64_t i = 0; i < n; ++i) { /* a drifting activation with per-column scales */
      seed = seed * 1664525u + 1013904223u;
      const float z = ((float)(seed >> 8) / 16777216.0f - 0.5f) * 2.0f;
      cur[i] += (t == 1 ? 1.0f : 0.1f) * z * (1.0f + (float)(i % cols) / (float)cols);
      hx[i] = to_bf16(cur[i]);
    }
    cudaMemcpyAsync(dx, hx, 2 * n, cudaMemcpyHostToDevice, st);
    CHECK(cc_allgather_step(layer, dx, st));
    if (t == 1) {
      CHECK(cc_warmup_step(CC_WITH_FEEDBACK, rows, cols, dx, CC_BF16, base, fb, body, CC_BF16, rec, st));
      CHECK(cc_decode_step(CC_RAW, 0, rows, cols, 0, body, CC_BF16, rbase, st));
    } else {
      CHECK(cc_encode_step(CC_QUANT2, CC_WITH_FEEDBACK, CC_SCALE_RANK1, rows, cols, dx, CC_BF16, base, fb, body, ws,
                           wsb, rec, st));
      CHECK(cc_decode_step(CC_QUANT2, 1, rows, cols, 0, body, CC_F32, rbase, st));
    }
    cudaStreamSynchronize(st);
    int64_t nb = 0;
    const uint8_t *lbody = cc_allgather_body(layer, &nb);
    if (!same(lbody, body, (size_t)nb)) { fprintf(stderr, "body differs at step %d\n", t); return 3; }
    if (!same(cc_allgather_sender_base(layer), base, 4 * n)) { fprintf(stderr, "base differs at step %d\n", t); return 3; }
    if (!same(cc_allgather_reconstruction(layer), rbase, 4 * n)) { fprintf(stderr, "receiver differs at step %d\n", t); return 3; }
    if (!same(cc_allgather_reconstruction(layer), cc_allgather_sender_base(layer), 4 * n)) {
      fprintf(stderr, "receiver != sender at step %d\n", t);
      return 3;
    }
  }
  CHECK(cc_allgather_destroy(layer));
  CHECK(cc_comm_destroy(comm));
  printf("exchange_demo ok: %d steps of [%lldx%lld] quant2bit through cc_allgather_step, %lld launches\n", steps,
         (long long)rows, (long long)cols, (long long)cc_launch_count());
  return 0;
}
