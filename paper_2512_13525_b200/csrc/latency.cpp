// latency.cpp — the MoE-layer latency model, calibrated to the measured
// layer.
//
// The reference prices one MoE instance as (src/latency.cpp:17-24)
//     t = t_launch + max(A * W_e / beta, F(b) / pi),
//     W_e = 2 * d_h * d_e * bpp   (ModelSpec::expert_weight_bytes, types.hpp:42-44)
//     F(b) = 2 * b * d_h * d_e
// and a layer as the max over instances with activated experts (:26-32).  The
// device runs a SwiGLU expert (three matrices: 1.5x the bytes and 3x the FLOPs
// per routed row), and its weight streaming and tensor work overlap only in
// part around the ridge.  janus_latency_model generalises the form:
//     t = t_launch + (mem^p + comp^p)^(1/p),
//     mem = A * matrices * d_h * d_e * bpp / beta,  comp = b * 2 * flop_matrices * d_h * d_e / pi
// p = infinity (p <= 0) is the reference's max; matrices = 2, flop_matrices = 1
// its accounting (SwiGLU: 3 and 3).
// janus_latency_fit fits (t_launch, beta, pi, p) to measured (A, b, t) points
// by Nelder–Mead on the mean squared relative error, in log parameters.
#include <algorithm>
#include <array>
#include <cmath>
#include <vector>

#include "janus_b200.h"

namespace {

double instance_time(const janus_latency_model &m, double A, double b, int d_h, int d_e) {
  const double mem = A * m.matrices * (double)d_h * d_e * m.bytes_per_param / m.hbm_bandwidth;
  const double comp = b * 2.0 * m.flop_matrices * (double)d_h * d_e / m.peak_flops;
  if (m.p <= 0 || m.p >= 64) return m.t_launch + std::max(mem, comp);
  const double hi = std::max(mem, comp);
  if (hi <= 0) return m.t_launch;
  // scaled p-norm (no overflow for large p)
  const double s = std::pow(mem / hi, m.p) + std::pow(comp / hi, m.p);
  return m.t_launch + hi * std::pow(s, 1.0 / m.p);
}

struct Fit {
  const int n;
  const int32_t *A;
  const int64_t *b;
  const double *t;
  int d_h, d_e;
  janus_latency_model base;
  janus_latency_model at(const std::array<double, 4> &x) const {
    janus_latency_model m = base;
    m.t_launch = std::exp(x[0]);
    m.hbm_bandwidth = std::exp(x[1]);
    m.peak_flops = std::exp(x[2]);
    m.p = 1.0 + std::exp(x[3]);  // p in (1, inf)
    return m;
  }
  double cost(const std::array<double, 4> &x) const {
    const janus_latency_model m = at(x);
    double c = 0;
    for (int i = 0; i < n; ++i) {
      const double r = (instance_time(m, A[i], (double)b[i], d_h, d_e) - t[i]) / t[i];
      c += r * r;
    }
    return c / n;
  }
};

// Nelder–Mead on 4 parameters (restarted once from its own optimum).
std::array<double, 4> minimise(const Fit &f, std::array<double, 4> x0) {
  using V = std::array<double, 4>;
  for (int restart = 0; restart < 2; ++restart) {
    std::array<V, 5> s;
    std::array<double, 5> c;
    s[0] = x0;
    for (int i = 0; i < 4; ++i) {
      s[i + 1] = x0;
      s[i + 1][i] += 0.5;
    }
    for (int i = 0; i < 5; ++i) c[i] = f.cost(s[i]);
    for (int it = 0; it < 4000; ++it) {
      std::array<int, 5> o = {0, 1, 2, 3, 4};
      std::sort(o.begin(), o.end(), [&](int a, int b) { return c[a] < c[b]; });
      if (c[o[4]] - c[o[0]] < 1e-14) break;
      V cen{};
      for (int k = 0; k < 4; ++k)
        for (int j = 0; j < 4; ++j) cen[j] += s[o[k]][j] / 4;
      auto lerp = [&](double a) {
        V v;
        for (int j = 0; j < 4; ++j) v[j] = cen[j] + a * (s[o[4]][j] - cen[j]);
        return v;
      };
      const V xr = lerp(-1.0);
      const double cr = f.cost(xr);
      if (cr < c[o[0]]) {
        const V xe = lerp(-2.0);
        const double ce = f.cost(xe);
        if (ce < cr) {
          s[o[4]] = xe;
          c[o[4]] = ce;
        } else {
          s[o[4]] = xr;
          c[o[4]] = cr;
        }
      } else if (cr < c[o[3]]) {
        s[o[4]] = xr;
        c[o[4]] = cr;
      } else {
        const V xc = lerp(0.5);
        const double cc = f.cost(xc);
        if (cc < c[o[4]]) {
          s[o[4]] = xc;
          c[o[4]] = cc;
        } else {
          for (int k = 1; k < 5; ++k) {
            for (int j = 0; j < 4; ++j) s[o[k]][j] = s[o[0]][j] + 0.5 * (s[o[k]][j] - s[o[0]][j]);
            c[o[k]] = f.cost(s[o[k]]);
          }
        }
      }
    }
    int best = 0;
    for (int i = 1; i < 5; ++i)
      if (c[i] < c[best]) best = i;
    x0 = s[best];
  }
  return x0;
}

}  // namespace

extern "C" {

double janus_latency_instance(const janus_latency_model *m, int activated_experts,
                              int64_t routed_tokens, int d_hidden, int d_expert) {
  if (!m || activated_experts <= 0) return 0.0;
  return instance_time(*m, activated_experts, (double)routed_tokens, d_hidden, d_expert);
}

double janus_latency_layer(const janus_latency_model *m, int num_instances, const int32_t *load,
                           const int64_t *routed_tokens, int d_hidden, int d_expert) {
  double worst = 0;  // latency.cpp:26-32: max over the instances that have work
  for (int g = 0; g < num_instances; ++g)
    if (load[g] > 0)
      worst = std::max(worst, janus_latency_instance(m, load[g], routed_tokens[g], d_hidden,
                                                     d_expert));
  return worst;
}

janus_status janus_latency_fit(int n, const int32_t *activated, const int64_t *routed_tokens,
                               const double *seconds, int d_hidden, int d_expert,
                               janus_latency_model *model, double *mean_abs_rel_err) {
  if (n < 4 || !activated || !routed_tokens || !seconds || !model || d_hidden <= 0 ||
      d_expert <= 0 || model->matrices <= 0 || model->bytes_per_param <= 0 ||
      model->flop_matrices <= 0 ||
      model->hbm_bandwidth <= 0 || model->peak_flops <= 0)
    return JANUS_EINVAL;
  for (int i = 0; i < n; ++i)
    if (!(seconds[i] > 0) || activated[i] <= 0) return JANUS_EINVAL;
  Fit f{n, activated, routed_tokens, seconds, d_hidden, d_expert, *model};
  const double p0 = model->p > 1 && model->p < 64 ? model->p : 4.0;
  std::array<double, 4> x = {std::log(std::max(model->t_launch, 1e-6)),
                             std::log(model->hbm_bandwidth), std::log(model->peak_flops),
                             std::log(p0 - 1.0)};
  x = minimise(f, x);
  *model = f.at(x);
  if (mean_abs_rel_err) {
    double e = 0;
    for (int i = 0; i < n; ++i)
      e += std::fabs(instance_time(*model, activated[i], (double)routed_tokens[i], d_hidden,
                                   d_expert) - seconds[i]) / seconds[i];
    *mean_abs_rel_err = e / n;
  }
  return JANUS_OK;
}

}  // extern "C"
