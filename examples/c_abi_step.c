/*
 * One policy-loss step through librl's C ABI from plain C — no Python, no torch.
 *
 *   c_abi_step DIR NUM_PROMPTS GROUP_SIZE
 *
 * DIR is an input artifact (synth/artifact.py: hidden.bf16, w_vocab.bf16, targets.i32,
 * infer_logprobs.f32, rewards.f32, rollout_offsets.i32, loss_mask.u8; T, H, V are derived
 * from the file sizes and NUM_PROMPTS * GROUP_SIZE rollouts). The program uploads W_vocab,
 * runs rl_policy_loss_fwd_bwd_hostio (per-step inputs from host memory, advantages by
 * rl_group_advantages on the device; Eq.1 / Eq.2 with alpha = 0.5,
 * beta = 5, guard 1e-5, L470-472) and writes DIR/c_d_hidden.f32 ([T, H], from the bf16
 * output), DIR/c_d_w_vocab.f32 ([V, H]) and DIR/c_report.txt (loss and counters).
 * tests/test_gpu_c_abi.py compares them with the fp64 oracle's files in the same DIR.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rl.h"

static void* read_file(const char* dir, const char* name, size_t* bytes) {
  char path[4096];
  snprintf(path, sizeof(path), "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) {
    fprintf(stderr, "cannot open %s\n", path);
    exit(2);
  }
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc(n > 0 ? (size_t)n : 1);
  if (n > 0 && fread(p, 1, (size_t)n, f) != (size_t)n) {
    fprintf(stderr, "short read %s\n", path);
    exit(2);
  }
  fclose(f);
  *bytes = (size_t)n;
  return p;
}

static void write_file(const char* dir, const char* name, const void* p, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof(path), "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f || fwrite(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "cannot write %s\n", path);
    exit(2);
  }
  fclose(f);
}

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                       \
      return 3;                                                                      \
    }                                                                                \
  } while (0)
#define RL(x)                                                                        \
  do {                                                                               \
    rl_status s_ = (x);                                                              \
    if (s_ != RL_OK) {                                                               \
      fprintf(stderr, "%s: %s (%s)\n", #x, rl_status_string(s_), rl_last_error_message()); \
      return 4;                                                                      \
    }                                                                                \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 4) {
    fprintf(stderr, "usage: %s DIR NUM_PROMPTS GROUP_SIZE\n", argv[0]);
    return 1;
  }
  const char* dir = argv[1];
  const int32_t np = atoi(argv[2]), g = atoi(argv[3]), R = np * g;
  size_t nb_h, nb_w, nb_t, nb_i, nb_r, nb_o, nb_m;
  uint16_t* hidden = (uint16_t*)read_file(dir, "hidden.bf16", &nb_h);
  uint16_t* w = (uint16_t*)read_file(dir, "w_vocab.bf16", &nb_w);
  int32_t* targets = (int32_t*)read_file(dir, "targets.i32", &nb_t);
  float* infer = (float*)read_file(dir, "infer_logprobs.f32", &nb_i);
  float* rewards = (float*)read_file(dir, "rewards.f32", &nb_r);
  int32_t* offsets = (int32_t*)read_file(dir, "rollout_offsets.i32", &nb_o);
  uint8_t* loss_mask = (uint8_t*)read_file(dir, "loss_mask.u8", &nb_m);
  const int64_t T = (int64_t)(nb_t / 4);
  const int64_t H = T > 0 ? (int64_t)(nb_h / 2 / (size_t)T) : 0;
  const int64_t V = H > 0 ? (int64_t)(nb_w / 2 / (size_t)H) : 0;
  if (T <= 0 || H <= 0 || V <= 0 || nb_r != (size_t)R * 4 || nb_o != (size_t)(R + 1) * 4) {
    fprintf(stderr, "inconsistent artifact sizes\n");
    return 1;
  }
  double D = 0;
  for (int64_t t = 0; t < T; ++t) D += loss_mask[t];  /* R5: the loss tokens of the batch */

  rl_lm_shape shape;
  memset(&shape, 0, sizeof(shape));
  shape.T = T;
  shape.H = H;
  shape.V_local = V;
  shape.V_global = V;
  shape.inv_temperature = 1.0f;
  rl_loss_params params;
  memset(&params, 0, sizeof(params));
  params.alpha = 0.5f;
  params.beta = 5.0f;
  params.guard_threshold = 1e-5f;
  params.num_rollouts = R;
  params.loss_denominator = D;

  /* model state on the device: W_vocab in, the two gradients out */
  uint16_t *d_w = NULL, *d_dh = NULL;
  float* d_dw = NULL;
  rl_loss_report* d_rep = NULL;
  void* ws = NULL;
  const size_t ws_bytes = rl_workspace_bytes_hostio(&shape, R, 0);
  if (ws_bytes == 0) {
    fprintf(stderr, "rl_workspace_bytes_hostio: %s\n", rl_last_error_message());
    return 4;
  }
  CK(cudaMalloc((void**)&d_w, nb_w));
  CK(cudaMalloc((void**)&d_dh, (size_t)T * H * 2));
  CK(cudaMalloc((void**)&d_dw, (size_t)V * H * 4));
  CK(cudaMalloc((void**)&d_rep, sizeof(rl_loss_report)));
  CK(cudaMalloc(&ws, ws_bytes));
  CK(cudaMemcpy(d_w, w, nb_w, cudaMemcpyHostToDevice));

  rl_loss_outputs out;
  memset(&out, 0, sizeof(out));
  out.report = d_rep;
  out.d_hidden = d_dh;
  out.d_w_vocab = d_dw;
  rl_loss_report rep;
  RL(rl_policy_loss_fwd_bwd_hostio(&shape, &params, g, hidden, d_w, targets, infer, rewards, offsets, loss_mask,
                                   &out, &rep, ws, ws_bytes, NULL));

  uint16_t* dh_bf = (uint16_t*)malloc((size_t)T * H * 2);
  float* dh = (float*)malloc((size_t)T * H * 4);
  float* dw = (float*)malloc((size_t)V * H * 4);
  CK(cudaMemcpy(dh_bf, d_dh, (size_t)T * H * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(dw, d_dw, (size_t)V * H * 4, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < T * H; ++i) {
    const uint32_t b = (uint32_t)dh_bf[i] << 16;
    memcpy(&dh[i], &b, 4);
  }
  write_file(dir, "c_d_hidden.f32", dh, (size_t)T * H * 4);
  write_file(dir, "c_d_w_vocab.f32", dw, (size_t)V * H * 4);
  char text[1024];
  const int n = snprintf(text, sizeof(text),
                         "loss %.17g\nmismatch_kl_sum %.17g\nkept_tokens %u\nmasked_low %u\nmasked_high %u\n"
                         "guarded_rollouts %u\nguarded_tokens %u\nnonfinite_inputs %u\nbad_targets %u\n"
                         "bad_offsets %u\nlaunches %d\n",
                         rep.loss, rep.mismatch_kl_sum, rep.kept_tokens, rep.masked_low, rep.masked_high,
                         rep.guarded_rollouts, rep.guarded_tokens, rep.nonfinite_inputs, rep.bad_targets,
                         rep.bad_offsets, rl_last_launch_count());
  write_file(dir, "c_report.txt", text, (size_t)n);
  printf("T %lld H %lld V %lld loss %.9g kept %u guarded %u launches %d\n", (long long)T, (long long)H,
         (long long)V, rep.loss, rep.kept_tokens, rep.guarded_rollouts, rl_last_launch_count());
  cudaFree(d_w);
  cudaFree(d_dh);
  cudaFree(d_dw);
  cudaFree(d_rep);
  cudaFree(ws);
  return 0;
}
