// latsum_b200/latsum.hpp — header-only C++ mirror of the reference's hot-path API
// (/root/reference/proj/include/latsum) over the C ABI in <latsum_b200.h>.
//
// Same names, argument meaning and exception types as the reference:
//   build_reference_canonical   reference.hpp:95-153
//   assembled_sum_canonical     lattice_sum.hpp:198-223  (LatticeGeometry on lattice_grid)
//   defected_sum                lattice_sum.hpp:339-400  (canonical branch)
//   sublattice_union_sum        lattice_sum.hpp:411-465
//   rhosvd                      rank_reduction.hpp:176-218
//   TuckerTensor::entry/to_dense tucker.hpp:38-54,172-178
//   CanonicalTensor::entry/weights/factor canonical.hpp:63-70
// Errors: std::invalid_argument, WindowOverflowError (std::out_of_range, .mode()),
// std::length_error, NotImplementedError, std::runtime_error (CUDA / cuSOLVER / NCCL).
// Storage is plain std::vector<double> in Eigen's column-major layout, so an Eigen
// build maps every buffer without copies (Eigen::Map<MatrixXd>(v.data(), rows, cols)).
#pragma once
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <map>
#include <optional>
#include <ostream>
#include <set>
#include <variant>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "latsum_b200.h"

namespace latsum {

using Index = int64_t;
using Dims3 = std::array<Index, 3>;
using Int3 = std::array<int, 3>;

class WindowOverflowError : public std::out_of_range {
 public:
  WindowOverflowError(const std::string& m, int mode) : std::out_of_range(m), mode_(mode) {}
  int mode() const { return mode_; }

 private:
  int mode_;
};

class NotImplementedError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace b200 {

inline void throw_status(int st, const std::string& msg) {
  switch (st) {
    case LATSUM_OK: return;
    case LATSUM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LATSUM_ERR_WINDOW_OVERFLOW: {
      int mode = 0;
      const auto p = msg.find("mode ");
      if (p != std::string::npos) mode = std::atoi(msg.c_str() + p + 5);
      throw WindowOverflowError(msg, mode);
    }
    case LATSUM_ERR_LENGTH: throw std::length_error(msg);
    case LATSUM_ERR_NOT_IMPLEMENTED: throw NotImplementedError(msg);
    default: throw std::runtime_error(msg);
  }
}

// One CUDA device / stream / cuSOLVER handle (latsum_ctx); one per host thread.
class Context {
 public:
  explicit Context(int device = 0) {
    latsum_ctx* c = nullptr;
    if (latsum_ctx_create(device, &c) != LATSUM_OK)
      throw std::runtime_error("latsum_ctx_create: no CUDA device (there is no CPU fallback)");
    ctx_.reset(c);
  }
  latsum_ctx* get() const { return ctx_.get(); }
  void check(int st) const {
    if (st != LATSUM_OK) throw_status(st, latsum_last_error(ctx_.get()));
  }
  static Context& default_context() {
    thread_local Context c(0);
    return c;
  }

 private:
  struct Del {
    void operator()(latsum_ctx* c) const { latsum_ctx_destroy(c); }
  };
  std::unique_ptr<latsum_ctx, Del> ctx_;
};

}  // namespace b200

// kernel.hpp:37-152 restricted to the gauss-type primitives of the hot path.
struct KernelSpec {
  int family = LATSUM_NEWTON;
  double lambda = 0.0;
  bool operator==(const KernelSpec& o) const { return family == o.family && lambda == o.lambda; }
  std::string key() const {
    return family == LATSUM_YUKAWA ? "yukawa(" + std::to_string(lambda) + ")" : "newton";
  }
  static KernelSpec newton() { return {LATSUM_NEWTON, 0.0}; }
  static KernelSpec yukawa(double l) {
    if (!(l > 0.0)) throw std::invalid_argument("yukawa lambda must be positive");
    return {LATSUM_YUKAWA, l};
  }
};

// grid.hpp:41-97 (box widths b_l and even cell counts n_l; origin 0).
struct UniformGrid {
  std::array<double, 3> box{1, 1, 1};
  Dims3 n{2, 2, 2};
  static UniformGrid cubic(double b, Index n) { return {{b, b, b}, {n, n, n}}; }
  Index points(int l) const { return n[l]; }
  double mesh(int l) const { return box[l] / double(n[l]); }
};

// geometry.hpp:15-121 (the parts the hot path consumes).
enum class DefectKind { vacancy, impurity };
struct DefectSpec {
  std::vector<Int3> sites;
  DefectKind kind = DefectKind::vacancy;
  double charge = 0.0;
  std::optional<KernelSpec> kernel;  // impurities may carry their own kernel
  std::array<double, 3> grid_offset{0, 0, 0};
};
inline std::vector<int> default_active_set(int cells) {
  std::vector<int> k;
  for (int i = -(cells / 2); i <= (cells + 1) / 2 - 1; ++i) k.push_back(i);
  return k;
}
struct LatticeGeometry {
  Int3 cells{1, 1, 1};
  double cell_width = 1.0;
  double base_charge = 1.0;
  KernelSpec kernel = KernelSpec::newton();
  std::array<std::vector<int>, 3> active;  // empty = default K sets
  std::vector<DefectSpec> defects;
  std::vector<int> active_set(int mode) const {
    return active[mode].empty() ? default_active_set(cells[mode]) : active[mode];
  }
};
struct SublatticePlacement {
  LatticeGeometry geom;
  std::array<double, 3> offset_cells{0, 0, 0};
};

// lattice_sum.hpp:75-86
inline UniformGrid lattice_grid(const LatticeGeometry& g, Index n_per_cell) {
  if (n_per_cell < 2 || n_per_cell % 2 != 0)
    throw std::invalid_argument("lattice_grid: points per cell must be even and >= 2");
  UniformGrid grid;
  for (int l = 0; l < 3; ++l) {
    grid.box[l] = g.cell_width * double(g.cells[l]);
    grid.n[l] = n_per_cell * g.cells[l];
  }
  return grid;
}

struct TruncationSpec {  // rank_reduction.hpp:21-43
  std::optional<Dims3> ranks;
  std::optional<double> tolerance;
  int max_als_sweeps = 30;
  double als_stagnation_tol = 1e-8;
  static TruncationSpec fixed_ranks(Index a, Index b, Index c) {
    TruncationSpec s;
    s.ranks = Dims3{a, b, c};
    return s;
  }
  static TruncationSpec tol(double eps) {
    TruncationSpec s;
    s.tolerance = eps;
    return s;
  }
};

struct SpectralReport {  // rank_reduction.hpp:49-67
  std::array<std::vector<double>, 3> singular_values;
  Dims3 chosen_ranks{0, 0, 0};
  double bound_abs = 0, bound_rel = 0, weight_norm = 0, input_norm = 0, stability_constant = 0;
  bool stability_ok = false;
  std::array<bool, 3> tie_at_cutoff{false, false, false};
  double tail(int mode) const {
    double s = 0;
    for (size_t k = size_t(chosen_ranks[mode]); k < singular_values[mode].size(); ++k)
      s += singular_values[mode][k] * singular_values[mode][k];
    return std::sqrt(s);
  }
};

// Device-resident reference tensor (reference.hpp:65-80).
class ReferenceTensor {
 public:
  ReferenceTensor(b200::Context& ctx, latsum_reference* h, KernelSpec k, UniformGrid base, int M)
      : ctx_(&ctx), h_(h, latsum_reference_destroy), kernel(k), base_grid(base), M(M) {
    int r = 0;
    double c0 = 0, sh[2];
    latsum_reference_info(h, &r, &c0, sh);
    rank_ = r;
    step_constant = c0;
    shell_a = sh[0];
    shell_A = sh[1];
  }
  Index rank() const { return rank_; }
  std::vector<double> factor(int mode) const {  // canonical.factor(mode): 2N x R
    std::vector<double> f(size_t(2 * base_grid.n[mode]) * rank_);
    ctx_->check(latsum_reference_factor(ctx_->get(), h_.get(), mode, f.data()));
    return f;
  }
  std::vector<double> weights() const {
    std::vector<double> w(rank_);
    b200::throw_status(latsum_reference_weights(h_.get(), w.data()), "reference weights");
    return w;
  }
  latsum_reference* handle() const { return h_.get(); }
  b200::Context& ctx() const { return *ctx_; }

  KernelSpec kernel;
  UniformGrid base_grid;
  int M = 0;
  double step_constant = 0, shell_a = 0, shell_A = 0;

 private:
  b200::Context* ctx_;
  std::shared_ptr<latsum_reference> h_;
  Index rank_ = 0;
};

inline ReferenceTensor build_reference_canonical(const KernelSpec& kernel, const UniformGrid& grid,
                                                 int M, double step_constant = 0.0,
                                                 b200::Context& ctx = b200::Context::default_context()) {
  latsum_reference* h = nullptr;
  ctx.check(latsum_reference_build(ctx.get(), kernel.family, kernel.lambda, grid.n.data(),
                                   grid.box.data(), M, step_constant, &h));
  return ReferenceTensor(ctx, h, kernel, grid, M);
}

// Device-resident canonical tensor (canonical.hpp:19-202).
class CanonicalTensor {
 public:
  CanonicalTensor(b200::Context& ctx, latsum_canonical* h)
      : ctx_(&ctx), h_(h, latsum_canonical_destroy) {
    latsum_canonical_info(h, dims_.data(), &rank_, dict_.data(), &merged_);
  }
  const Dims3& dims() const { return dims_; }
  Index rank() const { return rank_; }
  std::vector<double> weights() const {
    std::vector<double> w(rank_);
    b200::throw_status(latsum_canonical_weights(h_.get(), w.data()), "canonical weights");
    return w;
  }
  std::vector<double> factor(int mode) const {  // N_l x M_c, column-major
    std::vector<double> f(size_t(dims_[mode]) * rank_);
    ctx_->check(latsum_canonical_factor(ctx_->get(), h_.get(), mode, f.data()));
    return f;
  }
  double entry(Index i, Index j, Index k) const {
    const int64_t p[3] = {i, j, k};
    double v = 0;
    ctx_->check(latsum_canonical_entries(ctx_->get(), h_.get(), p, 1, &v));
    return v;
  }
  latsum_canonical* handle() const { return h_.get(); }
  b200::Context& ctx() const { return *ctx_; }

 private:
  b200::Context* ctx_;
  std::shared_ptr<latsum_canonical> h_;
  Dims3 dims_{0, 0, 0}, dict_{0, 0, 0};
  Index rank_ = 0, merged_ = 0;
};

// Device-resident Tucker tensor (tucker.hpp:19-73).
class TuckerTensor {
 public:
  TuckerTensor(b200::Context& ctx, latsum_tucker* h) : ctx_(&ctx), h_(h, latsum_tucker_destroy) {
    latsum_tucker_info(h, dims_.data(), ranks_.data());
  }
  const Dims3& dims() const { return dims_; }
  const Dims3& ranks() const { return ranks_; }
  double entry(Index i, Index j, Index k) const {
    const int64_t p[3] = {i, j, k};
    double v = 0;
    ctx_->check(latsum_tucker_entries(ctx_->get(), h_.get(), p, 1, &v));
    return v;
  }
  std::vector<double> core() const {
    std::vector<double> c(size_t(ranks_[0]) * ranks_[1] * ranks_[2]);
    ctx_->check(latsum_tucker_core(ctx_->get(), h_.get(), c.data()));
    return c;
  }
  std::vector<double> factor(int mode) const {
    std::vector<double> f(size_t(dims_[mode]) * ranks_[mode]);
    ctx_->check(latsum_tucker_factor(ctx_->get(), h_.get(), mode, f.data()));
    return f;
  }
  latsum_tucker* handle() const { return h_.get(); }
  b200::Context& ctx() const { return *ctx_; }

 private:
  b200::Context* ctx_;
  std::shared_ptr<latsum_tucker> h_;
  Dims3 dims_{0, 0, 0}, ranks_{0, 0, 0};
};

// to_dense (tucker.hpp:172-178) with the reference's 1e7-entry guard.
inline std::vector<double> to_dense(const TuckerTensor& t, Index guard = 10'000'000) {
  const Dims3 d = t.dims();
  if (d[0] * d[1] * d[2] > guard)
    throw std::length_error("dense materialization of " + std::to_string(d[0] * d[1] * d[2]) +
                            " entries exceeds the guard limit " + std::to_string(guard));
  std::vector<double> out(size_t(d[0] * d[1] * d[2]));
  const int64_t lo[3] = {0, 0, 0}, hi[3] = {d[0], d[1], d[2]};
  if (!out.empty()) t.ctx().check(latsum_tucker_eval_box(t.ctx().get(), t.handle(), lo, hi, out.data()));
  return out;
}

namespace detail {
inline long lround_away(double x) { return std::lround(x); }

// Ordered product blocks for latsum_canonical_assemble_blocks: per block three shift lists
// (mesh units) and an additive charge; R terms per block, in block (add_concat) order.
struct Blocks {
  std::vector<int64_t> counts, shifts;
  std::vector<double> charges;
  void add(const std::array<std::vector<int64_t>, 3>& sh, double q) {
    for (int l = 0; l < 3; ++l) {
      counts.push_back(int64_t(sh[l].size()));
      shifts.insert(shifts.end(), sh[l].begin(), sh[l].end());
    }
    charges.push_back(q);
  }
  int64_t size() const { return int64_t(charges.size()); }
};

// lattice_sum.hpp:278-294: the per-mode sorted index sets if the sites are their full
// Cartesian product
inline std::optional<std::array<std::vector<int>, 3>> product_structure(const std::vector<Int3>& sites) {
  std::array<std::set<int>, 3> axes;
  for (const auto& s : sites)
    for (int l = 0; l < 3; ++l) axes[l].insert(s[l]);
  size_t prod = 1;
  for (int l = 0; l < 3; ++l) prod *= axes[l].size();
  if (prod != sites.size()) return std::nullopt;
  std::set<Int3> have(sites.begin(), sites.end());
  for (int a : axes[0])
    for (int b : axes[1])
      for (int c : axes[2])
        if (!have.count(Int3{a, b, c})) return std::nullopt;
  std::array<std::vector<int>, 3> out;
  for (int l = 0; l < 3; ++l) out[l].assign(axes[l].begin(), axes[l].end());
  return out;
}

// assembled_vector's active sets (lattice_sum.hpp:198-223, :444 offsets)
inline void add_lattice(Blocks& b, const LatticeGeometry& g, const std::array<double, 3>& off,
                        Index n) {
  std::array<std::vector<int64_t>, 3> sh;
  for (int l = 0; l < 3; ++l)
    for (int k : g.active_set(l))
      sh[l].push_back(int64_t(k) * n + lround_away(off[l] * double(n)));
  b.add(sh, g.base_charge);
}

// defect_cluster_canonical (lattice_sum.hpp:297-330): a product cluster is one assembled
// block at reference rank, any other cluster one window per site in site order; returns
// the number of blocks (the cluster's rank in units of R)
inline Index add_defect(Blocks& b, const DefectSpec& d, Index n) {
  std::array<long, 3> off;
  for (int l = 0; l < 3; ++l) off[l] = lround_away(d.grid_offset[l]);
  if (d.sites.size() > 1) {
    if (auto axes = product_structure(d.sites)) {
      std::array<std::vector<int64_t>, 3> sh;
      for (int l = 0; l < 3; ++l)
        for (int v : (*axes)[l]) sh[l].push_back(int64_t(v) * n + off[l]);
      b.add(sh, d.charge);
      return 1;
    }
  }
  for (const auto& s : d.sites) {  // defect_grid_shift (:159-164)
    std::array<std::vector<int64_t>, 3> sh;
    for (int l = 0; l < 3; ++l) sh[l].push_back(int64_t(s[l]) * n + off[l]);
    b.add(sh, d.charge);
  }
  return Index(d.sites.size());
}

inline Index active_cells(const LatticeGeometry& g) {
  Index c = 1;
  for (int l = 0; l < 3; ++l) c *= Index(g.active_set(l).size());
  return c;
}
}  // namespace detail

inline CanonicalTensor assemble(const ReferenceTensor& ref, const detail::Blocks& b) {
  b200::Context& ctx = ref.ctx();
  latsum_canonical* h = nullptr;
  ctx.check(latsum_canonical_assemble_blocks(ctx.get(), ref.handle(), b.size(), b.counts.data(),
                                             b.shifts.data(), b.charges.data(), &h));
  return CanonicalTensor(ctx, h);
}

// add_concat (canonical.hpp:94-110): a + b by concatenation, a's terms first
inline CanonicalTensor add_concat(const CanonicalTensor& a, const CanonicalTensor& b) {
  b200::Context& ctx = a.ctx();
  latsum_canonical* h = nullptr;
  ctx.check(latsum_canonical_concat(ctx.get(), a.handle(), b.handle(), &h));
  return CanonicalTensor(ctx, h);
}

// Rank-R canonical lattice sum + additive defects on the lattice_grid of `geom`
// (assembled_sum_canonical + defected_sum without truncation, in one assembly).
inline CanonicalTensor defected_sum(const ReferenceTensor& ref, const LatticeGeometry& geom,
                                    Index n_per_cell,
                                    const std::vector<SublatticePlacement>* subs = nullptr) {
  detail::Blocks b;
  if (subs && !subs->empty()) {
    for (const auto& s : *subs) detail::add_lattice(b, s.geom, s.offset_cells, n_per_cell);
  } else {
    detail::add_lattice(b, geom, {0, 0, 0}, n_per_cell);
  }
  for (const auto& d : geom.defects) detail::add_defect(b, d, n_per_cell);
  return assemble(ref, b);
}

inline CanonicalTensor assembled_sum_canonical(const ReferenceTensor& ref,
                                               const LatticeGeometry& geom, Index n_per_cell) {
  if (!geom.defects.empty())
    throw std::invalid_argument("assembled_sum_canonical: geometry carries defects; use defected_sum");
  return defected_sum(ref, geom, n_per_cell);
}

inline CanonicalTensor sublattice_union_sum(const std::vector<SublatticePlacement>& subs,
                                            const ReferenceTensor& ref,
                                            const LatticeGeometry& parent, Index n_per_cell) {
  if (subs.empty()) throw std::invalid_argument("sublattice_union_sum: no sublattices");
  LatticeGeometry p = parent;
  p.defects.clear();
  return defected_sum(ref, p, n_per_cell, &subs);
}

inline SpectralReport to_report(const latsum_spectral_report& rep, latsum_tucker* h) {
  SpectralReport out;
  for (int l = 0; l < 3; ++l) {
    out.singular_values[l].resize(size_t(rep.n_singular[l]));
    latsum_tucker_singular_values(h, l, out.singular_values[l].data());
    out.chosen_ranks[l] = rep.chosen_ranks[l];
    out.tie_at_cutoff[l] = rep.tie_at_cutoff[l] != 0;
  }
  out.bound_abs = rep.bound_abs;
  out.bound_rel = rep.bound_rel;
  out.weight_norm = rep.weight_norm;
  out.input_norm = rep.input_norm;
  out.stability_constant = rep.stability_constant;
  out.stability_ok = rep.stability_ok != 0;
  return out;
}

inline std::pair<TuckerTensor, SpectralReport> rhosvd(const CanonicalTensor& a,
                                                      const TruncationSpec& spec,
                                                      int deflate = LATSUM_DEFLATE_AUTO) {
  if (!spec.ranks && !spec.tolerance)
    throw std::invalid_argument("TruncationSpec: need ranks or tolerance");
  b200::Context& ctx = a.ctx();
  latsum_tucker* h = nullptr;
  latsum_spectral_report rep;
  ctx.check(latsum_rhosvd(ctx.get(), a.handle(), spec.ranks ? spec.ranks->data() : nullptr,
                          spec.tolerance.value_or(0.0), deflate, &h, &rep));
  TuckerTensor t(ctx, h);
  return {std::move(t), to_report(rep, h)};
}

// rank_reduction.hpp:280-306: rhosvd, ALS refinement (spec.max_als_sweeps,
// spec.als_stagnation_tol) and, tolerance-driven, shrink_core
inline std::pair<TuckerTensor, SpectralReport> canonical_to_tucker(const CanonicalTensor& a,
                                                                   const TruncationSpec& spec) {
  if (!spec.ranks && !spec.tolerance)
    throw std::invalid_argument("TruncationSpec: need ranks or tolerance");
  b200::Context& ctx = a.ctx();
  latsum_tucker* h = nullptr;
  latsum_spectral_report rep;
  ctx.check(latsum_canonical_to_tucker(ctx.get(), a.handle(), spec.ranks ? spec.ranks->data() : nullptr,
                                       spec.tolerance.value_or(0.0), spec.max_als_sweeps,
                                       spec.als_stagnation_tol, &h, &rep, nullptr));
  TuckerTensor t(ctx, h);
  return {std::move(t), to_report(rep, h)};
}

// ---- the reference's result-level interface (lattice_sum.hpp:38-69, :260-276, :339-465)

enum class Accumulation { sliding, ascending, compensated };
// lattice_sum.hpp:28-39.  sliding (default): uniformly strided shift lists are summed by the
// reference's recursion (lattice_sum.hpp:116-128) in its operation order, every other list
// directly; ascending: always directly; compensated: accepted, summed in the ascending order
// (latsum_ctx_set_accumulation).
struct SumOptions {
  Accumulation accumulation = Accumulation::sliding;
};
inline void apply(const SumOptions& o, b200::Context& ctx) {
  ctx.check(latsum_ctx_set_accumulation(ctx.get(), int(o.accumulation)));
}

struct Summand {  // lattice_sum.hpp:44-50
  std::string label;
  Index canonical_rank = 0;
  Index sites = 0;
};

struct LatticeSumResult {  // lattice_sum.hpp:52-69
  std::variant<CanonicalTensor, TuckerTensor> tensor;
  LatticeGeometry geometry;
  UniformGrid grid;
  std::vector<Summand> provenance;
  std::optional<SpectralReport> report;
  // the product blocks of the untruncated sum (defected_sum re-assembles base + clusters in
  // one device call instead of add_concat copies)
  std::shared_ptr<const detail::Blocks> blocks;
  bool is_canonical() const { return tensor.index() == 0; }
  const CanonicalTensor& canonical() const { return std::get<CanonicalTensor>(tensor); }
  const TuckerTensor& tucker_tensor() const { return std::get<TuckerTensor>(tensor); }
};

class ReferenceSet {  // lattice_sum.hpp:260-276
 public:
  void add(ReferenceTensor ref) { refs_.push_back(std::move(ref)); }
  const ReferenceTensor& find(const KernelSpec& kernel) const {
    for (const auto& r : refs_)
      if (r.kernel == kernel) return r;
    throw std::invalid_argument("no reference tensor built for kernel " + kernel.key());
  }
  bool has(const KernelSpec& kernel) const {
    for (const auto& r : refs_)
      if (r.kernel == kernel) return true;
    return false;
  }

 private:
  std::vector<ReferenceTensor> refs_;
};

// The base result cmd_sum builds for a rectangular lattice (commands.cpp:160-163).
inline LatticeSumResult assembled_sum_result(const ReferenceTensor& ref,
                                             const LatticeGeometry& geom,
                                             const SumOptions& opts = {}) {
  apply(opts, ref.ctx());
  LatticeGeometry rect = geom;
  rect.defects.clear();
  const Index n = ref.base_grid.n[0] / rect.cells[0];
  auto b = std::make_shared<detail::Blocks>();
  detail::add_lattice(*b, rect, {0, 0, 0}, n);
  auto can = assemble(ref, *b);
  LatticeSumResult out{std::move(can), rect, ref.base_grid, {}, std::nullopt, b};
  out.provenance.push_back({"assembled lattice sum", out.canonical().rank(), detail::active_cells(rect)});
  return out;
}

// defected_sum (lattice_sum.hpp:339-384), canonical branch: base + defect clusters in
// `defects` order, truncated by canonical_to_tucker when `spec` is set.  Clusters with the base
// kernel that come before any other kernel join the base's product blocks (one device assembly
// instead of add_concat copies); from the first cluster carrying its own kernel
// (DefectSpec.kernel, :301-303) on, every maximal run of clusters sharing a kernel is assembled
// against that kernel's reference tensor (refs.find) and added with add_concat, in order — the
// same terms in the same order as the reference's per-cluster add_concat loop (:372-374).
inline LatticeSumResult defected_sum(const LatticeSumResult& base,
                                     const std::vector<DefectSpec>& defects,
                                     const ReferenceSet& refs,
                                     const std::optional<TruncationSpec>& spec,
                                     const SumOptions& opts = {}) {
  if (defects.empty()) return base;
  apply(opts, base.canonical().ctx());
  if (!base.is_canonical())
    throw NotImplementedError("defected_sum: the GPU path sums canonical bases (the Tucker-format "
                              "route is out of scope)");
  for (const auto& d : defects) {
    if (d.sites.empty()) throw std::invalid_argument("defected_sum: defect with no sites");
    const KernelSpec k = d.kernel ? *d.kernel : base.geometry.kernel;
    if (!refs.has(k))
      throw std::invalid_argument("defected_sum: no reference tensor for kernel " + k.key());
  }
  const Index n = base.grid.n[0] / base.geometry.cells[0];
  LatticeSumResult out{base.tensor, base.geometry, base.grid, base.provenance, std::nullopt, nullptr};
  auto kernel_of = [&](const DefectSpec& d) { return d.kernel ? *d.kernel : base.geometry.kernel; };
  auto record = [&](const DefectSpec& d, Index blocks, const ReferenceTensor& ref) {
    out.provenance.push_back({d.kind == DefectKind::vacancy ? "vacancy cluster" : "impurity cluster",
                              blocks * ref.rank(), Index(d.sites.size())});
    out.geometry.defects.push_back(d);
  };
  size_t at = 0;
  std::optional<CanonicalTensor> total;
  if (base.blocks) {  // leading base-kernel clusters: re-assembled with the base in one call
    const ReferenceTensor& ref = refs.find(base.geometry.kernel);
    auto b = std::make_shared<detail::Blocks>(*base.blocks);
    for (; at < defects.size() && kernel_of(defects[at]) == base.geometry.kernel; ++at)
      record(defects[at], detail::add_defect(*b, defects[at], n), ref);
    total = assemble(ref, *b);
    if (at == defects.size()) out.blocks = b;  // still one block list: later calls may extend it
  } else {
    total = base.canonical();
  }
  while (at < defects.size()) {  // runs of clusters sharing a kernel
    const KernelSpec k = kernel_of(defects[at]);
    const ReferenceTensor& ref = refs.find(k);
    detail::Blocks b;
    for (; at < defects.size() && kernel_of(defects[at]) == k; ++at)
      record(defects[at], detail::add_defect(b, defects[at], n), ref);
    total = add_concat(*total, assemble(ref, b));
  }
  if (spec) {
    auto tr = canonical_to_tucker(*total, *spec);
    out.tensor = std::move(tr.first);
    out.report = std::move(tr.second);
  } else {
    out.tensor = std::move(*total);
  }
  return out;
}

// sublattice_union_sum (lattice_sum.hpp:411-465): one assembled block per sublattice
inline LatticeSumResult sublattice_union_sum(const std::vector<SublatticePlacement>& subs,
                                             const ReferenceTensor& ref,
                                             const LatticeGeometry& geometry,
                                             const std::optional<TruncationSpec>& spec,
                                             const SumOptions& opts = {}) {
  if (subs.empty()) throw std::invalid_argument("sublattice_union_sum: no sublattices");
  apply(opts, ref.ctx());
  const Index n = ref.base_grid.n[0] / geometry.cells[0];
  auto b = std::make_shared<detail::Blocks>();
  LatticeSumResult out{sublattice_union_sum(subs, ref, geometry, n), geometry, ref.base_grid, {},
                       std::nullopt, b};
  for (const auto& s : subs) {
    detail::add_lattice(*b, s.geom, s.offset_cells, n);
    out.provenance.push_back({"sublattice", ref.rank(), detail::active_cells(s.geom)});
  }
  if (spec) {
    auto tr = canonical_to_tucker(out.canonical(), *spec);
    out.tensor = std::move(tr.first);
    out.report = std::move(tr.second);
  }
  return out;
}

// report.cpp:28-46 write_spectral_report (the library's formatter: same text, byte for byte)
inline void write_spectral_report(std::ostream& os, const SpectralReport& r) {
  latsum_spectral_report c{};
  const double* sv[3];
  for (int l = 0; l < 3; ++l) {
    c.chosen_ranks[l] = r.chosen_ranks[l];
    c.tie_at_cutoff[l] = r.tie_at_cutoff[l] ? 1 : 0;
    c.n_singular[l] = int64_t(r.singular_values[l].size());
    sv[l] = r.singular_values[l].data();
  }
  c.bound_abs = r.bound_abs;
  c.bound_rel = r.bound_rel;
  c.weight_norm = r.weight_norm;
  c.input_norm = r.input_norm;
  c.stability_constant = r.stability_constant;
  c.stability_ok = r.stability_ok ? 1 : 0;
  const int64_t n = latsum_format_spectral_report(&c, sv, nullptr, 0);
  std::string buf(size_t(n) + 1, '\0');
  latsum_format_spectral_report(&c, sv, &buf[0], n + 1);
  os.write(buf.data(), n);
}

// report.cpp:48-73 write_provenance, for a result described by its grid, geometry cells,
// tensor ranks and summands (label, canonical rank, sites)
inline void write_provenance(std::ostream& os, const Dims3& grid, const Dims3& cells,
                             const std::optional<Dims3>& tucker_ranks, Index canonical_rank,
                             const std::vector<Summand>& summands,
                             const std::optional<SpectralReport>& report, std::uint64_t seed,
                             const std::vector<std::string>& extra_lines = {}) {
  latsum_provenance p{};
  p.seed = seed;
  for (int l = 0; l < 3; ++l) {
    p.grid[l] = grid[l];
    p.cells[l] = cells[l];
  }
  p.format = tucker_ranks ? 1 : 0;
  p.rank = canonical_rank;
  if (tucker_ranks)
    for (int l = 0; l < 3; ++l) p.ranks[l] = (*tucker_ranks)[l];
  std::vector<const char*> labels, extra;
  std::vector<int64_t> ranks, sites;
  for (const auto& s : summands) {
    labels.push_back(s.label.c_str());
    ranks.push_back(s.canonical_rank);
    sites.push_back(s.sites);
  }
  for (const auto& e : extra_lines) extra.push_back(e.c_str());
  p.nsummands = int64_t(summands.size());
  p.labels = labels.data();
  p.summand_ranks = ranks.data();
  p.summand_sites = sites.data();
  if (report) {
    p.has_report = 1;
    p.bound_abs = report->bound_abs;
    p.bound_rel = report->bound_rel;
  }
  p.nextra = int64_t(extra.size());
  p.extra = extra.data();
  const int64_t n = latsum_format_provenance(&p, nullptr, 0);
  std::string buf(size_t(n) + 1, '\0');
  latsum_format_provenance(&p, &buf[0], n + 1);
  os.write(buf.data(), n);
}

// report.cpp:48-73 with the reference's signature
inline void write_provenance(std::ostream& os, const LatticeSumResult& result, std::uint64_t seed,
                             const std::vector<std::string>& extra_lines = {}) {
  const Dims3 cells{result.geometry.cells[0], result.geometry.cells[1], result.geometry.cells[2]};
  std::optional<Dims3> tr;
  Index rank = 0;
  if (result.is_canonical()) rank = result.canonical().rank();
  else tr = result.tucker_tensor().ranks();
  write_provenance(os, result.grid.n, cells, tr, rank, result.provenance, result.report, seed,
                   extra_lines);
}

}  // namespace latsum
