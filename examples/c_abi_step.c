/* c_abi_step.c -- the stage from plain C through include/attn_softmax.h (no
 * Python, no PyTorch): allocate with the CUDA runtime, fill deterministic
 * inputs, run attn_softmax_fwd_bwd once, print the loss and a gradient norm.
 * Build (plain C): gcc -std=c99 -o c_abi_step examples/c_abi_step.c -Iinclude \
 *          -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -lm \
 *          -Lpaper_1909_00562_b200/lib -lattnsm -Wl,-rpath,<lib dir>  */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "attn_softmax.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
      return 1;                                                                 \
    }                                                                           \
  } while (0)
#define AK(x)                                                                   \
  do {                                                                          \
    attn_status_t s_ = (x);                                                     \
    if (s_ != ATTN_OK) {                                                        \
      fprintf(stderr, "%s: status %d: %s\n", #x, (int)s_, attn_last_error());  \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

static uint16_t to_bf16(float f) {   /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static float lcg(uint32_t* s) {      /* uniform in [-1, 1) */
  *s = *s * 1664525u + 1013904223u;
  return (float)(*s >> 8) / (float)(1u << 23) - 1.f;
}
static int fill(void* dev, size_t n, float scale, uint32_t seed) {
  uint16_t* h = (uint16_t*)malloc(n * 2);
  for (size_t i = 0; i < n; ++i) h[i] = to_bf16(scale * lcg(&seed));
  cudaError_t e = cudaMemcpy(dev, h, n * 2, cudaMemcpyHostToDevice);
  free(h);
  return e == cudaSuccess ? 0 : 1;
}

int main(int argc, char** argv) {
  const int B = 16, N = 24, M = 20, d = 256, V = 4000;
  attn_shape_t s = {B, N, M, d, V, ATTN_BF16};
  printf("%s\n", attn_version());
  const size_t T = (size_t)B * N;
  void *Hd, *He, *Wc, *Wo, *dHd, *dHe, *ws;
  float *loss, *dWc, *dWo;
  int32_t* ids;
  CK(cudaMalloc(&Hd, T * d * 2));
  CK(cudaMalloc(&He, (size_t)B * M * d * 2));
  CK(cudaMalloc(&Wc, (size_t)d * 2 * d * 2));
  CK(cudaMalloc(&Wo, (size_t)V * d * 2));
  CK(cudaMalloc(&dHd, T * d * 2));
  CK(cudaMalloc(&dHe, (size_t)B * M * d * 2));
  CK(cudaMalloc((void**)&dWc, (size_t)d * 2 * d * 4));
  CK(cudaMalloc((void**)&dWo, (size_t)V * d * 4));
  CK(cudaMalloc((void**)&loss, 4));
  CK(cudaMalloc((void**)&ids, T * 4));
  if (fill(Hd, T * d, 0.35f, 1) || fill(He, (size_t)B * M * d, 0.35f, 2) ||
      fill(Wc, (size_t)d * 2 * d, 0.1f, 3) || fill(Wo, (size_t)V * d, 0.1f, 4))
    return 1;
  int32_t* hid = (int32_t*)malloc(T * 4);
  uint32_t seed = 5;
  for (size_t t = 0; t < T; ++t) hid[t] = 4 + (int32_t)((lcg(&seed) + 1.f) * 0.5f * (V - 5));
  CK(cudaMemcpy(ids, hid, T * 4, cudaMemcpyHostToDevice));
  int32_t src[16], tgt[16];
  int total = 0;
  for (int b = 0; b < B; ++b) {
    src[b] = 1 + (b * 7) % M;
    tgt[b] = (b * 5) % (N + 1);
    total += tgt[b];
  }
  const size_t wsb = attn_softmax_workspace_size(&s);
  if (!wsb) { fprintf(stderr, "workspace: %s\n", attn_last_error()); return 1; }
  CK(cudaMalloc(&ws, wsb));
  AK(attn_softmax_fwd_bwd(&s, Hd, He, src, tgt, ids, Wc, Wo, NULL, 1.f / (float)total, loss, dHd,
                          dHe, dWc, dWo, NULL, ws, wsb, NULL, 0));
  CK(cudaDeviceSynchronize());
  float hl;
  CK(cudaMemcpy(&hl, loss, 4, cudaMemcpyDeviceToHost));
  float* g = (float*)malloc((size_t)V * d * 4);
  CK(cudaMemcpy(g, dWo, (size_t)V * d * 4, cudaMemcpyDeviceToHost));
  double nrm = 0, colsum = 0;
  for (size_t i = 0; i < (size_t)V * d; ++i) nrm += (double)g[i] * g[i];
  for (int v = 0; v < V; ++v) colsum += g[(size_t)v * d];   /* column 0 of dW_out sums to ~0 */
  printf("loss %.6f (ln V = %.6f)  |dW_out| %.6e  sum_v dW_out[v,0] %.3e\n", hl, log((double)V),
         sqrt(nrm), colsum);
  /* a documented error path: W_alpha without dW_alpha */
  attn_status_t st = attn_softmax_fwd_bwd(&s, Hd, He, src, tgt, ids, Wc, Wo, Wc, 1.f, loss, dHd,
                                          dHe, dWc, dWo, NULL, ws, wsb, NULL, 0);
  printf("W_alpha without dW_alpha -> status %d (%s)\n", (int)st, attn_last_error());
  return (st == ATTN_ERR_INVALID_ARG && isfinite(hl) && fabs(hl - log((double)V)) < 1.0) ? 0 : 2;
}
