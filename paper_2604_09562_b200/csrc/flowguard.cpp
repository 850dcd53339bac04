// FlowGuard lane router (NEXT-2): PAPER.md §3.3 eq:flowguard_score, eq:overload_detection /
// eq:overload_score, eq:fallback_selection, Alg. 2; readings DESIGN.md
// R25-R28. Host scalar code behind include/sv.h: picks the decode lane for an incoming request.
#include <math.h>
#include <string.h>

#include "../../include/sv.h"

namespace {

bool valid_cfg(const sv_route_config* c) {
  if (!c || !(c->tau > 0.0) || !(c->q_max >= 1.0) || c->staleness_ms < 0) return false;
  double s = 0.0;
  for (int j = 0; j < 4; ++j) {
    if (!(c->alpha[j] >= 0.0)) return false;
    s += c->alpha[j];
  }
  return fabs(s - 1.0) <= 1e-9;
}

bool frac(double x) { return x >= 0.0 && x <= 1.0; }

}  // namespace

extern "C" {

void sv_route_default_config(sv_route_config* c) {
  if (!c) return;
  memset(c, 0, sizeof(*c));
  c->alpha[0] = 0.4;
  c->alpha[1] = 0.1;
  c->alpha[2] = 0.3;
  c->alpha[3] = 0.2;
  c->tau = 0.85;
  c->q_max = 100.0;
  c->staleness_ms = 1000;
}

sv_status sv_route_select(const sv_route_config* c, int32_t n, const sv_lane_metrics* m, const double* live_queue,
                          int64_t now_ms, int32_t* chosen, double* scores, uint8_t* flags, int32_t* used_fallback) {
  if (!valid_cfg(c) || n < 1 || !m || !chosen) return SV_EINVAL;
  for (int i = 0; i < n; ++i) {
    const double q = live_queue ? live_queue[i] : m[i].queue_depth;
    if (!frac(m[i].cache_hit) || !frac(m[i].mem_util) || !frac(m[i].active_load) || !(q >= 0.0)) return SV_EINVAL;
  }
  int best = -1;
  double best_s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double q = live_queue ? live_queue[i] : m[i].queue_depth;
    const bool stale = now_ms - m[i].timestamp_ms > c->staleness_ms;             // R27
    const double omega = (100.0 * m[i].mem_util) / 100.0 + 2.0 * (q / c->q_max);  // eq:overload_score, R25
    const bool over = omega > c->tau;                                            // eq:overload_detection
    double s = NAN;
    if (!stale && !over) {
      const double qw = fmin(q / c->q_max, 1.0);                                 // R26
      s = c->alpha[0] * m[i].cache_hit + c->alpha[1] * (1.0 - m[i].mem_util) + c->alpha[2] * (1.0 - qw) +
          c->alpha[3] * (1.0 - m[i].active_load);                                // eq:flowguard_score
      if (best < 0 || s > best_s) {                                              // argmax, lowest index on ties
        best = i;
        best_s = s;
      }
    }
    if (scores) scores[i] = s;
    if (flags) flags[i] = (uint8_t)((over ? SV_ROUTE_OVERLOADED : 0) | (stale ? SV_ROUTE_STALE : 0));
  }
  int fb = 0;
  if (best < 0) {                                                                // eq:fallback_selection
    fb = 1;
    best = 0;
    for (int i = 1; i < n; ++i) {
      const double qi = live_queue ? live_queue[i] : m[i].queue_depth;
      const double qb = live_queue ? live_queue[best] : m[best].queue_depth;
      if (qi < qb) best = i;
    }
  }
  *chosen = best;
  if (used_fallback) *used_fallback = fb;
  return SV_OK;
}

}  // extern "C"
