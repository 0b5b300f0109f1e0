// Host-side rules of the hot path (no GPU): sinc quadrature, the calibrated
// step-constant sweep and the reference shell.  They are microseconds of scalar
// work that the reference also runs on the host; keeping
// them on the host with FMA contraction off (-ffp-contract=off) makes the nodes
// t_k and weights a_k bit-identical to the reference's libm arithmetic, which
// the 1e-12 directional parity of stage 1 depends on.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <limits>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "latsum_b200.h"

namespace {

// Persistent host workers for the step-constant sweep: spawning a thread per candidate
// cost more than the sweep itself (~15 us per std::thread, 53 candidates, every call).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  // f(0) .. f(n-1), the caller participating; returns when all have run
  void run(int n, const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(run_mu_);  // one sweep at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      f_ = &f;
      n_ = n;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return done_ == n_; });
    f_ = nullptr;
  }

 private:
  HostPool() {
    const int nt = std::max(0, std::min(31, int(std::thread::hardware_concurrency()) - 1));
    for (int i = 0; i < nt; ++i)
      threads_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> g(mu_);
            cv_.wait(g, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
          }
          work();
        }
      });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void work() {  // claim (f, i) under the lock: a claimed task keeps its run() alive
    for (;;) {
      const std::function<void(int)>* f;
      int i;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!f_ || next_ >= n_) return;
        f = f_;
        i = next_++;
      }
      (*f)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* f_ = nullptr;
  int n_ = 0, done_ = 0, next_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

double transform_weight(int family, double lambda, double t) {
  // quadrature.hpp:73-85: p(z) = int_0^inf w(t) exp(-z^2 t^2) dt
  const double c = 2.0 / std::sqrt(M_PI);
  if (family == LATSUM_NEWTON) return c;
  if (t == 0.0) return 0.0;
  const double kap = lambda / 2.0;
  return c * std::exp(-(kap * kap) / (t * t));
}

double closed_form(int family, double lambda, double r) {
  // kernel.hpp:154-158
  return family == LATSUM_NEWTON ? 1.0 / r : std::exp(-lambda * r) / r;
}

void sinc_rule(int family, double lambda, int M, double c0, double A, double* t, double* a) {
  // quadrature.hpp:155-163: u_k = (k - M) h_M, t_k = sinh(u_k)/A,
  // a_k = (h_M/2) w(|t_k|) cosh(u_k)/A, h_M = C0 log(M)/M
  const double hM = c0 * std::log(double(M)) / double(M);
  for (int k = 0; k < 2 * M + 1; ++k) {
    const double u = (double(k) - double(M)) * hM;
    const double tk = std::sinh(u) / A;
    t[k] = tk;
    a[k] = 0.5 * hM * transform_weight(family, lambda, std::abs(tk)) * std::cosh(u) / A;
  }
}

double max_pointwise_rel(int family, double lambda, const double* t, const double* a, int R,
                         double lo, double hi, int npts) {
  // quadrature.hpp:217-234 (shell_error) with separable_eval (:191-201) at (z,0,0)
  const double la = std::log(lo), lA = std::log(hi);
  double worst = 0.0;
  for (int i = 0; i < npts; ++i) {
    const double z = std::exp(la + (lA - la) * double(i) / double(npts - 1));
    // separable_eval at (z, 0, 0): the two zero coordinates contribute
    // exp(-s*0*0) = exp(-0) = 1 exactly, so only the first factor is evaluated
    // (bit-identical to the three-factor product).
    double sum = 0.0;
    for (int k = 0; k < R; ++k) {
      const double s = t[k] * t[k];
      double prod = a[k];
      prod *= std::exp(-s * z * z);
      sum += prod;
    }
    const double exact = closed_form(family, lambda, z);
    worst = std::fmax(worst, std::abs(1.0 * sum - exact) / std::abs(exact));
  }
  return worst;
}

}  // namespace

extern "C" {

int latsum_build_quadrature(int family, double lambda, int M, double step_constant,
                            double shell_a, double shell_A, double* nodes, double* weights) {
  if (family != LATSUM_NEWTON && family != LATSUM_YUKAWA) return LATSUM_ERR_NOT_IMPLEMENTED;
  if (M < 2 || !(shell_a > 0.0) || !(shell_A > shell_a) || !(step_constant > 0.0))
    return LATSUM_ERR_INVALID_ARGUMENT;
  if (family == LATSUM_YUKAWA && !(lambda > 0.0)) return LATSUM_ERR_INVALID_ARGUMENT;
  sinc_rule(family, lambda, M, step_constant, shell_A, nodes, weights);
  return LATSUM_OK;
}

double latsum_default_step_constant(int family, double lambda, int M, double shell_a,
                                    double shell_A, int npts) {
  // quadrature.hpp:238-269: 53 candidates base*(0.5 + 1.3 i/52),
  // base = asinh(2.5 A/a)/log M; first strict minimum of the finite errors.
  if (npts <= 1) npts = 320;
  // The 53 candidates are independent: evaluate them on host threads, then pick the
  // first strict minimum in candidate order exactly as the sequential sweep does.
  const double base = std::asinh(2.5 * (shell_A / shell_a)) / std::log(double(M));
  constexpr int kCand = 53;
  double c0s[kCand], errs[kCand];
  for (int i = 0; i < kCand; ++i) c0s[i] = base * (0.5 + 1.3 * double(i) / 52.0);
  const std::function<void(int)> cand = [&](int i) {
    std::vector<double> t(2 * M + 1), a(2 * M + 1);
    sinc_rule(family, lambda, M, c0s[i], shell_A, t.data(), a.data());
    errs[i] = max_pointwise_rel(family, lambda, t.data(), a.data(), 2 * M + 1, shell_a, shell_A, npts);
  };
  HostPool::get().run(kCand, cand);
  double best = std::numeric_limits<double>::infinity();
  double best_c0 = c0s[0];
  for (int i = 0; i < kCand; ++i)
    if (std::isfinite(errs[i]) && errs[i] < best) {
      best = errs[i];
      best_c0 = c0s[i];
    }
  return best_c0;
}

void latsum_reference_shell(const int64_t N[3], const double box[3], double shell[2]) {
  // reference.hpp:84-93 on the doubled grid: mesh h_l = 2b_l / 2N_l, width 2b_l
  double hmin = (2.0 * box[0]) / double(2 * N[0]);
  double bmax = 0.0;
  for (int l = 0; l < 3; ++l) {
    hmin = std::fmin(hmin, (2.0 * box[l]) / double(2 * N[l]));
    bmax = std::fmax(bmax, 2.0 * box[l]);
  }
  shell[0] = hmin;
  shell[1] = std::sqrt(3.0) * bmax / 2.0;
}

void latsum_verify_probes(uint64_t seed, const int64_t dims[3], int64_t n, int64_t* probes) {
  // commands.cpp:254-260 cmd_verify's probe stream, the same standard-library objects in the
  // same order: one std::mt19937_64(seed), three uniform_int_distribution<Index>(0, d_l - 1),
  // (i, j, k) drawn per probe
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int64_t> di(0, dims[0] - 1), dj(0, dims[1] - 1), dk(0, dims[2] - 1);
  for (int64_t p = 0; p < n; ++p) {
    probes[3 * p] = di(rng);
    probes[3 * p + 1] = dj(rng);
    probes[3 * p + 2] = dk(rng);
  }
}

}  // extern "C"
