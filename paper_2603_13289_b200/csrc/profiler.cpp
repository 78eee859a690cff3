// profiler.cpp -- host side of the offline layer profiler: layer curves
// (similarity + adjacent-layer Spearman), curve averaging and the start / end
// / detection scans that turn the averaged curve into a LayerProfile. The
// per-instance work (captures, prefills, token deviations) runs on the device
// (rk_profile_model, engine.cpp). Each function restates the reference's
// arithmetic in the same order (double, left to right), so results are
// bit-identical.
#include "profiler.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <string>

namespace rk {
namespace prof {
namespace {

// average_ranks (metrics.cpp:48-64): stable order by value, ties share the mean rank.
std::vector<double> average_ranks(const std::vector<double>& x) {
  const size_t n = x.size();
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return x[a] < x[b]; });
  std::vector<double> ranks(n);
  for (size_t i = 0; i < n;) {
    size_t j = i;
    while (j + 1 < n && x[order[j + 1]] == x[order[i]]) ++j;
    const double r = 0.5 * ((double)i + (double)j) + 1.0;
    for (size_t k = i; k <= j; ++k) ranks[order[k]] = r;
    i = j + 1;
  }
  return ranks;
}

// spearman (metrics.cpp:173-195); returns degenerate (rho 0) for constant input.
double spearman(const std::vector<double>& x, const std::vector<double>& y, bool* degenerate) {
  if (x.size() != y.size()) raise(RK_ERR_INVALID_ARGUMENT, "spearman: length mismatch");
  if (x.size() < 2) raise(RK_ERR_INVALID_ARGUMENT, "spearman: need at least 2 samples");
  const std::vector<double> rx = average_ranks(x), ry = average_ranks(y);
  const double n = (double)x.size();
  double mx = 0.0, my = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    mx += rx[i];
    my += ry[i];
  }
  mx /= n;
  my /= n;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    const double dx = rx[i] - mx, dy = ry[i] - my;
    sxy += dx * dy;
    sxx += dx * dx;
    syy += dy * dy;
  }
  *degenerate = sxx == 0.0 || syy == 0.0;
  return *degenerate ? 0.0 : sxy / std::sqrt(sxx * syy);
}

size_t argmin_first(const std::vector<double>& s) {
  size_t best = 0;
  for (size_t i = 1; i < s.size(); ++i)
    if (s[i] < s[best]) best = i;
  return best;
}

// find_start_layer (profiler.cpp:49-57)
size_t start_layer(const std::vector<double>& s, const rk_profiler_params& p) {
  validate_params(p);
  if (s.size() < 6) raise(RK_ERR_INVALID_ARGUMENT, "find_start_layer: curve shorter than 6");
  for (size_t l = argmin_first(s); l-- > 0;)
    if (s[l] >= p.tau_start) return l;
  return 0;
}

// find_end_layer (profiler.cpp:59-93): the first window of `consecutive`
// layers past the minimum that sits above the tail baseline with steps under
// lambda * tail sigma.
size_t end_layer(const std::vector<double>& s, const rk_profiler_params& p, bool* fallback) {
  validate_params(p);
  const size_t L = s.size();
  if (L < p.tail_layers + 2) raise(RK_ERR_INVALID_ARGUMENT, "find_end_layer: curve shorter than tail_layers + 2");
  double mu = 0.0;
  for (size_t l = L - p.tail_layers; l < L; ++l) mu += s[l];
  mu /= (double)p.tail_layers;
  double var = 0.0;
  for (size_t l = L - p.tail_layers; l < L; ++l) var += (s[l] - mu) * (s[l] - mu);
  var /= (double)p.tail_layers;
  const double sigma = std::sqrt(var), baseline = mu - sigma, max_step = p.stability_lambda * sigma;
  const size_t l_min = argmin_first(s);
  for (size_t l = std::max(l_min + p.min_rise, l_min + 1); l + p.consecutive <= L; ++l) {
    bool ok = true;
    for (size_t w = l; w < l + p.consecutive && ok; ++w) {
      const double step = std::abs(s[w] - s[w - 1]);
      const bool stable = sigma > 0.0 ? step < max_step : step == 0.0;
      ok = s[w] >= baseline && stable;
    }
    if (ok) {
      *fallback = false;
      return l;
    }
  }
  *fallback = true;
  return L - 1;
}

// find_detection_layer (profiler.cpp:95-121): one layer after the first
// concave turn of the adjacent-layer correlation curve inside (l_start, l_end].
size_t detection_layer(const std::vector<double>& rho, size_t l_start, size_t l_end, const rk_profiler_params& p,
                       bool* fallback) {
  validate_params(p);
  if (l_start >= l_end) raise(RK_ERR_INVALID_ARGUMENT, "find_detection_layer: requires l_start < l_end");
  if (rho.size() <= l_end) raise(RK_ERR_INVALID_ARGUMENT, "find_detection_layer: rho not defined up to l_end");
  auto alpha = [&](size_t l) { return rho[l] - 2.0 * rho[l - 1] + rho[l - 2]; };
  for (size_t l = std::max<size_t>(l_start + 2, p.first_negative_alpha ? 3 : 4); l <= l_end; ++l) {
    const bool hit = p.first_negative_alpha ? alpha(l) < 0.0 : (alpha(l - 1) > 0.0 && alpha(l) < 0.0);
    if (hit) {
      *fallback = false;
      return std::min(l + 1, l_end);
    }
  }
  *fallback = true;
  return l_start + 1;
}

uint64_t splitmix_next(uint64_t& state) {  // metrics.cpp:246-251
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

}  // namespace

void validate_params(const rk_profiler_params& p) {
  if (!(p.tau_start > 0.0 && p.tau_start <= 1.0))
    raise(RK_ERR_INVALID_ARGUMENT, "profiler params: tau_start must be in (0, 1]");
  if (p.tail_layers < 2) raise(RK_ERR_INVALID_ARGUMENT, "profiler params: tail_layers must be >= 2");
  if (!(p.stability_lambda > 0.0)) raise(RK_ERR_INVALID_ARGUMENT, "profiler params: stability_lambda must be > 0");
  if (p.consecutive < 1) raise(RK_ERR_INVALID_ARGUMENT, "profiler params: consecutive must be >= 1");
  if (p.min_rise < 1) raise(RK_ERR_INVALID_ARGUMENT, "profiler params: min_rise must be >= 1");
}

void validate_calib(const rk_two_stage_config& c) {
  if (c.instances == 0) raise(RK_ERR_SCHEMA, "two-stage config: instances must be >= 1");
  if (c.segment_len == 0) raise(RK_ERR_SCHEMA, "two-stage config: segment_len must be >= 1");
  if (c.stage1_prefix_min == 0 || c.stage1_prefix_min > c.stage1_prefix_max || c.stage2_prefix_min == 0 ||
      c.stage2_prefix_min > c.stage2_prefix_max)
    raise(RK_ERR_SCHEMA, "two-stage config: bad prefix length range");
}

Curve layer_curve(const double* dev, size_t n, size_t L) {  // make_layer_curve (metrics.cpp:191-213)
  if (n == 0) raise(RK_ERR_INVALID_ARGUMENT, "layer_similarity: empty segment");
  Curve c;
  c.s.assign(L, 0.0);
  for (size_t l = 0; l < L; ++l) {  // layer_similarity (metrics.cpp:162-171)
    double acc = 0.0;
    for (size_t j = 0; j < n; ++j) acc += 1.0 - dev[j * L + l];
    c.s[l] = acc / (double)n;
  }
  c.rho.assign(L, std::numeric_limits<double>::quiet_NaN());
  c.deg.assign(L, 1);
  std::vector<double> prev(n), cur(n);
  for (size_t l = 1; l < L; ++l) {
    if (n < 2) {
      c.rho[l] = 0.0;
      continue;
    }
    for (size_t j = 0; j < n; ++j) {
      prev[j] = dev[j * L + l - 1];
      cur[j] = dev[j * L + l];
    }
    bool degenerate = false;
    c.rho[l] = spearman(prev, cur, &degenerate);
    c.deg[l] = degenerate;
  }
  return c;
}

Curve average(const std::vector<Curve>& curves) {  // average_curves (metrics.cpp:215-238)
  if (curves.empty()) raise(RK_ERR_INVALID_ARGUMENT, "average_curves: no curves");
  const size_t L = curves[0].s.size();
  Curve a;
  a.s.assign(L, 0.0);
  a.rho.assign(L, std::numeric_limits<double>::quiet_NaN());
  a.deg.assign(L, 1);
  for (const Curve& c : curves) {
    if (c.s.size() != L) raise(RK_ERR_INVALID_ARGUMENT, "average_curves: layer mismatch");
    for (size_t l = 0; l < L; ++l) a.s[l] += c.s[l];
  }
  for (size_t l = 0; l < L; ++l) a.s[l] /= (double)curves.size();
  for (size_t l = 1; l < L; ++l) {
    double acc = 0.0;
    bool all = true;
    for (const Curve& c : curves) {
      acc += c.deg[l] ? 0.0 : c.rho[l];
      all = all && c.deg[l];
    }
    a.rho[l] = acc / (double)curves.size();
    a.deg[l] = all;
  }
  return a;
}

rk_profile_result from_curve(const Curve& c, const rk_profiler_params& p, std::vector<double>* curve_rho) {
  validate_params(p);
  const size_t L = c.s.size();
  if (L < std::max<size_t>(6, p.tail_layers + 2))
    raise(RK_ERR_INVALID_ARGUMENT, "profile_from_curve: too few layers for the scans");
  std::vector<double> crho(L > 1 ? L - 1 : 0, 0.0);
  for (size_t l = 1; l < L; ++l) crho[l - 1] = c.deg[l] ? 0.0 : c.rho[l];
  rk_profile_result r{};
  r.l_start = start_layer(c.s, p);
  bool fb = false;
  r.l_end = end_layer(c.s, p, &fb);
  r.end_fallback = fb;
  std::vector<double> rho_by_layer(L, 0.0);
  for (size_t l = 1; l < L; ++l) rho_by_layer[l] = crho[l - 1];
  r.l_det = detection_layer(rho_by_layer, r.l_start, r.l_end, p, &fb);
  r.det_fallback = fb;
  if (!(r.l_start <= r.l_det && r.l_det <= r.l_end && r.l_end < L))  // LayerProfile::validate
    raise(RK_ERR_SCHEMA, "layer profile violates l_start <= l_det <= l_end < num_layers (" +
                             std::to_string(r.l_start) + ", " + std::to_string(r.l_det) + ", " +
                             std::to_string(r.l_end) + ") for " + std::to_string(L) + " layers");
  if (curve_rho) *curve_rho = crho;
  return r;
}

std::vector<int32_t> synthetic_tokens(uint64_t seed, uint64_t salt, size_t count, size_t vocab) {
  uint64_t state = seed ^ (salt * 0x9e3779b97f4a7c15ull + 0x1234567ull);  // metrics.cpp:255-263
  std::vector<int32_t> out(count);
  for (auto& t : out) t = (int32_t)(splitmix_next(state) % vocab);
  return out;
}

size_t pick_length(uint64_t seed, uint64_t salt, size_t lo, size_t hi) {  // metrics.cpp:265-269
  if (hi <= lo) return lo;
  uint64_t state = seed ^ (salt * 0xd1b54a32d192ed03ull + 0xabcdull);
  return lo + (size_t)(splitmix_next(state) % (hi - lo + 1));
}

}  // namespace prof
}  // namespace rk
