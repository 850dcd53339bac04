// SpecuStream depth controller (NEXT-1): PAPER.md §3.5, Alg. 4 "SpecuStream Adaptation"
// (PAPER.md:374-391), readings DESIGN.md R21-R24. Host scalar code behind include/sv.h; the
// lane feeds it from its acceptance counters (a7) and applies the depth to its next verify.
#include <math.h>
#include <string.h>

#include "../../include/sv.h"

namespace {

bool valid(const sv_spec_config* c) {
  return c && c->h >= 1 && c->h <= SV_SPEC_MAX_H && c->d_min >= 1.0 && c->d_min <= c->d_base &&
         c->d_base <= c->d_max && c->gamma >= 0.0 && c->tau_target > 0.0 && c->micro_batch_numerator > 0.0 &&
         (c->projection_source == 0 || c->projection_source == 1);
}

double mean(const double* x, int n) {   // j = 0 .. h-1 in order
  double s = 0.0;
  for (int j = 0; j < n; ++j) s += x[j];
  return s / n;
}

}  // namespace

extern "C" {

void sv_spec_default_config(sv_spec_config* c) {
  if (!c) return;
  memset(c, 0, sizeof(*c));
  c->d_base = 5.0;
  c->gamma = 5.0;
  c->d_min = 2.0;
  c->d_max = 20.0;
  c->h = 10;
  c->projection_source = 0;
  c->tau_target = 400.0;
  c->micro_batch_numerator = 80.0;
}

sv_status sv_spec_reset(const sv_spec_config* c, sv_flow_state* st) {
  if (!valid(c) || !st) return SV_EINVAL;
  memset(st, 0, sizeof(*st));
  st->tau_recent = c->tau_target;
  return SV_OK;
}

sv_status sv_spec_adapt(const sv_spec_config* c, const sv_flow_state* in, double a, double l, double t,
                        sv_spec_plan* plan, sv_flow_state* out) {
  if (!valid(c) || !in || !plan || !out) return SV_EINVAL;
  if (in->idx < 0 || in->idx >= c->h || !(in->tau_recent >= 0.0)) return SV_EINVAL;
  if (!(a >= 0.0 && a <= 1.0) || !(l >= 0.0 && l <= 1.0) || !(t >= 0.0)) return SV_EINVAL;
  const int h = c->h;
  double f[SV_SPEC_MAX_H];
  memcpy(f, in->f, sizeof(double) * h);
  const double tau_old = in->tau_recent;
  // eq:acceptance_gradient: delta against the buffer before the write, then circular write
  const double delta = a - mean(f, h);
  f[in->idx] = delta;
  const int idx = (in->idx + 1) % h;
  // eq:flow_magnitude over the buffer after the write
  double af[SV_SPEC_MAX_H];
  for (int j = 0; j < h; ++j) af[j] = fabs(f[j]);
  const double mag = mean(af, h);
  const double scale = fmax(1.0, c->tau_target / fmax(t, 1.0));       // eq:throughput_scaling
  const double adj = 1.0 - fmin(l, 0.9);                               // eq:load_adaptation
  const double raw = c->d_base + (a * mag * c->gamma) * adj * scale;   // eq:optimal_depth
  const double clipped = fmin(fmax(raw, c->d_min), c->d_max);          // eq:depth_clipping
  const int depth = (int)floor(clipped + 0.5);                         // R21: token count
  int micro = (int)floor(c->micro_batch_numerator / depth);            // eq:microbatch_size
  if (micro < 1) micro = 1;
  const double src = c->projection_source == 0 ? t : tau_old;          // R22
  const double t_proj = src * (1.0 + a * 0.5);
  const double tau_new = 0.9 * tau_old + 0.1 * t_proj;                 // eq_exponential_smoothing
  plan->depth = depth;
  plan->micro_batch = micro;
  plan->projected = t_proj;
  plan->raw_depth = raw;
  plan->delta = delta;
  plan->mag = mag;
  plan->scale = scale;
  plan->adj = adj;
  if (out != in) memcpy(out, in, sizeof(*out));
  memcpy(out->f, f, sizeof(double) * h);
  out->idx = idx;
  out->tau_recent = tau_new;
  return SV_OK;
}

sv_status sv_spec_step(const sv_spec_config* c, const sv_flow_state* in, const sv_lane_stats* s0,
                       const sv_lane_stats* s1, double seconds, int32_t active, int32_t max_batch,
                       sv_spec_plan* plan, sv_flow_state* out) {
  if (!s0 || !s1 || !(seconds > 0.0) || max_batch < 1 || active < 0 || active > max_batch) return SV_EINVAL;
  if (s1->drafted < s0->drafted || s1->accepted < s0->accepted || s1->emitted < s0->emitted) return SV_EINVAL;
  const double drafted = (double)(s1->drafted - s0->drafted);
  const double a = drafted > 0.0 ? (double)(s1->accepted - s0->accepted) / drafted : 0.0;
  const double t = (double)(s1->emitted - s0->emitted) / seconds;
  const double l = (double)active / (double)max_batch;
  return sv_spec_adapt(c, in, a, l, t, plan, out);
}

}  // extern "C"
