// TEST INFRASTRUCTURE (oracle/): a C ABI over the REFERENCE'S OWN headers, compiled where they
// lie under /root/reference/proj/include (never copied), against the Eigen stand-in in
// oracle/shim (Eigen is absent from this image).  The library built from this file,
// oracle/_ref/liblatsum_ref.so, is the reference itself run here: tests use it to pin the CPU
// restatement (oracle/latsum_oracle.cpp, oracle.py) and the CUDA path to reference outputs.
// Every function below only marshals arrays in and out of the reference calls it names:
//   build_reference_canonical   reference.hpp:95-153
//   lattice_grid                lattice_sum.hpp:75-86
//   assembled_sum_canonical     lattice_sum.hpp:198-223
//   sublattice_union_sum        lattice_sum.hpp:411-465
//   defected_sum                lattice_sum.hpp:339-384
//   rhosvd / canonical_to_tucker  rank_reduction.hpp:176-218, 280-306
//   oracle_entry                lattice_sum.hpp:656-672
//   CanonicalTensor::entry / TuckerTensor::entry  canonical.hpp:63-70, tucker.hpp:38-54
//   write_spectral_report / write_provenance  src/report.cpp:28-73 (compiled from the reference's src/)
//   write_tensor / read_tensor  src/tensor_io.cpp (compiled from the reference's src/)
//   cmd_sum / cmd_verify  src/commands.cpp:108-177, 200-284 (compiled from the reference's src/;
//                         its reference cache is stubbed "never cached" by ref_nocache.cpp)
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it.
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <optional>
#include <string>
#include <vector>

#include "latsum/commands.hpp"
#include "latsum/lattice_sum.hpp"
#include "latsum/rank_reduction.hpp"
#include "latsum/reference.hpp"
#include "latsum/report.hpp"
#include "latsum/tensor_io.hpp"

using namespace latsum;

namespace {

struct Handle {
  LatticeGeometry geom;
  Index n_per_cell = 0;
  ReferenceTensor<double> ref;
  ReferenceSet<double> refs;
  std::optional<CanonicalTensor<double>> canonical;
  std::vector<Summand> provenance;
  LatticeGeometry out_geometry;  // the sum's geometry (parent cells + the defects added)
  std::vector<SublatticePlacement> placements;
  int M = 0;
  std::vector<std::pair<int, double>> defect_kernels;  // per DefectSpec: (family or -1, lambda)
  std::vector<GridSource<double>> sources;
  std::optional<TuckerTensor<double>> tucker;
  std::optional<SpectralReport<double>> report;
  std::string error;
};

thread_local std::string g_error;

template <typename Fn>
int guarded(Handle* h, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const WindowOverflowError& e) {
    (h ? h->error : g_error) = e.what();
    return 3;
  } catch (const NotImplementedError& e) {
    (h ? h->error : g_error) = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    (h ? h->error : g_error) = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    (h ? h->error : g_error) = e.what();
    return 2;
  } catch (const std::exception& e) {
    (h ? h->error : g_error) = e.what();
    return 9;
  }
}

KernelSpec make_kernel(int family, double lam) {
  return family == 0 ? KernelSpec::newton() : KernelSpec::yukawa(lam);
}

void copy_matrix(const MatrixX<double>& m, double* out) {
  if (out) std::memcpy(out, m.data(), sizeof(double) * size_t(m.rows() * m.cols()));
}

}  // namespace

extern "C" {

const char* lref_last_error(void* hp) {
  return hp ? static_cast<Handle*>(hp)->error.c_str() : g_error.c_str();
}

// geometry (cells, n_per_cell, cell_width, base charge, optional active K sets) + the kernel's
// reference tensor on the doubled grid; C0 <= 0 runs the reference's calibration sweep
void* lref_create(int family, double lam, int M, const int* cells, int n_per_cell,
                  double cell_width, double base_charge, double C0, const int* active,
                  const int* n_active) {
  auto h = std::make_unique<Handle>();
  const int rc = guarded(nullptr, [&] {
    h->geom.cells = {cells[0], cells[1], cells[2]};
    h->geom.cell_width = cell_width;
    h->geom.base_charge = base_charge;
    h->geom.kernel = make_kernel(family, lam);
    if (active && n_active) {
      const int* p = active;
      for (int l = 0; l < 3; ++l) {
        h->geom.active[l].assign(p, p + n_active[l]);
        p += n_active[l];
      }
    }
    h->n_per_cell = n_per_cell;
    h->M = M;
    h->geom.validate();
    const UniformGrid<double> grid = lattice_grid<double>(h->geom, n_per_cell);
    ReferenceOptions opts;
    opts.step_constant = C0;
    h->ref = build_reference_canonical<double>(h->geom.kernel, grid, M, opts);
    h->refs.add(h->ref);
  });
  return rc == 0 ? h.release() : nullptr;
}

void lref_destroy(void* hp) { delete static_cast<Handle*>(hp); }

// out[0..2] = 2N_l, out[3] = R, out[4..6] = N_l
int lref_ref_info(void* hp, int64_t* out, double* C0, double* shell) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    for (int l = 0; l < 3; ++l) {
      out[l] = h->ref.grid.points(l);
      out[4 + l] = h->ref.base_grid.points(l);
    }
    out[3] = h->ref.canonical.rank();
    if (C0) *C0 = h->ref.step_constants.at(0);
    if (shell) {
      shell[0] = h->ref.shell.a;
      shell[1] = h->ref.shell.A;
    }
  });
}

int lref_ref_copy(void* hp, double* f0, double* f1, double* f2, double* weights, double* nodes,
                  double* qweights) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    double* f[3] = {f0, f1, f2};
    for (int l = 0; l < 3; ++l) copy_matrix(h->ref.canonical.factor(l), f[l]);
    const Index r = h->ref.canonical.rank();
    if (weights) std::memcpy(weights, h->ref.canonical.weights().data(), sizeof(double) * size_t(r));
    const auto& rule = h->ref.expansion.terms.at(0).rule;
    if (nodes) std::memcpy(nodes, rule.nodes.data(), sizeof(double) * size_t(rule.size()));
    if (qweights) std::memcpy(qweights, rule.weights.data(), sizeof(double) * size_t(rule.size()));
  });
}

// The canonical lattice sum.  n_sub == 0: assembled_sum_canonical over the geometry's active
// sets; else sublattice_union_sum over n_sub rectangular sublattices (cells, offset_cells).
// Then defected_sum with n_def clusters: def_nsites[d] sites each (flattened in def_sites),
// charge, grid_offset (mesh units), kind (0 vacancy, 1 impurity).  accumulation: 0 sliding,
// 1 ascending, 2 compensated.
int lref_sum(void* hp, int n_sub, const int* sub_cells, const double* sub_offsets, int n_def,
             const int* def_nsites, const int* def_sites, const double* def_charge,
             const double* def_goff, const int* def_kind, int accumulation) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    SumOptions opts;
    opts.accumulation = accumulation == 0   ? Accumulation::sliding
                        : accumulation == 1 ? Accumulation::ascending
                                            : Accumulation::compensated;
    LatticeSumResult<double> base;
    h->sources.clear();
    h->placements.clear();
    if (n_sub == 0) {
      base.tensor = assembled_sum_canonical(h->ref, h->geom, opts);
      base.geometry = h->geom;
      base.grid = h->ref.base_grid;
      base.provenance.push_back({"assembled lattice sum", h->ref.canonical.rank(), Dims3{0, 0, 0},
                                 Index(active_cells(h->geom).size())});
      h->sources = enumerate_sources<double>(h->geom, h->n_per_cell);
    } else {
      std::vector<SublatticePlacement> subs;
      for (int s = 0; s < n_sub; ++s) {
        SublatticePlacement p;
        p.geom = h->geom;
        p.geom.active = {};
        p.geom.cells = {sub_cells[3 * s], sub_cells[3 * s + 1], sub_cells[3 * s + 2]};
        p.offset_cells = Array3<double>(sub_offsets[3 * s], sub_offsets[3 * s + 1],
                                        sub_offsets[3 * s + 2]);
        for (const auto& cell : active_cells(p.geom)) {
          GridSource<double> g;
          for (int l = 0; l < 3; ++l)
            g.shift[l] = long(cell[l]) * long(h->n_per_cell) +
                         std::lround(p.offset_cells[l] * double(h->n_per_cell));
          g.weight = h->geom.base_charge;
          g.kernel = h->geom.kernel;
          h->sources.push_back(g);
        }
        subs.push_back(std::move(p));
      }
      base = sublattice_union_sum<double>(subs, h->ref, h->geom, std::nullopt, opts);
      h->placements = subs;
    }
    std::vector<DefectSpec> defects;
    const int* site = def_sites;
    for (int d = 0; d < n_def; ++d) {
      DefectSpec spec;
      for (int s = 0; s < def_nsites[d]; ++s, site += 3) spec.sites.push_back({site[0], site[1], site[2]});
      spec.kind = def_kind && def_kind[d] ? DefectKind::impurity : DefectKind::vacancy;
      spec.charge = def_charge[d];
      if (def_goff)
        spec.grid_offset = Array3<double>(def_goff[3 * d], def_goff[3 * d + 1], def_goff[3 * d + 2]);
      if (size_t(d) < h->defect_kernels.size() && h->defect_kernels[size_t(d)].first >= 0) {
        // DefectSpec.kernel (geometry.hpp:26): the cluster carries its own kernel; its reference
        // tensor joins the ReferenceSet (same grid, same M), as cmd_sum does (commands.cpp:168-172)
        spec.kernel = make_kernel(h->defect_kernels[size_t(d)].first, h->defect_kernels[size_t(d)].second);
        if (!h->refs.has(*spec.kernel))
          h->refs.add(build_reference_canonical<double>(*spec.kernel, h->ref.base_grid, h->M, ReferenceOptions{}));
      }
      for (const auto& s : spec.sites) {
        GridSource<double> g;
        g.shift = detail::defect_grid_shift(s, spec.grid_offset, h->n_per_cell);
        g.weight = spec.charge;
        g.kernel = spec.kernel ? *spec.kernel : h->geom.kernel;
        h->sources.push_back(g);
      }
      defects.push_back(std::move(spec));
    }
    LatticeSumResult<double> out = defected_sum<double>(base, defects, h->refs, std::nullopt, opts);
    h->canonical = out.canonical();
    h->provenance = out.provenance;
    h->out_geometry = out.geometry;
    h->tucker.reset();
    h->report.reset();
  });
}

// per-DefectSpec kernels for the next lref_sum: family[d] < 0 keeps the base kernel
int lref_set_defect_kernels(void* hp, int n, const int* family, const double* lam) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    h->defect_kernels.clear();
    for (int d = 0; d < n; ++d) h->defect_kernels.emplace_back(family[d], lam[d]);
  });
}

int lref_canonical_info(void* hp, int64_t* rank, int64_t* n_summands) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (!h->canonical) throw std::invalid_argument("no canonical sum built");
    *rank = h->canonical->rank();
    if (n_summands) *n_summands = int64_t(h->provenance.size());
  });
}

// summand s: label into buf (NUL-terminated, <= cap), canonical rank and site count
int lref_summand(void* hp, int s, char* buf, int cap, int64_t* rank, int64_t* sites) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    const Summand& sm = h->provenance.at(size_t(s));
    std::strncpy(buf, sm.label.c_str(), size_t(cap - 1));
    buf[cap - 1] = 0;
    *rank = sm.canonical_rank;
    *sites = sm.sites;
  });
}

int lref_canonical_copy(void* hp, double* f0, double* f1, double* f2, double* weights) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (!h->canonical) throw std::invalid_argument("no canonical sum built");
    double* f[3] = {f0, f1, f2};
    for (int l = 0; l < 3; ++l) copy_matrix(h->canonical->factor(l), f[l]);
    if (weights)
      std::memcpy(weights, h->canonical->weights().data(), sizeof(double) * size_t(h->canonical->rank()));
  });
}

// mode 0: rhosvd, 1: canonical_to_tucker.  eps > 0: tolerance; ranks != null: fixed ranks.
int lref_reduce(void* hp, int mode, double eps, const int64_t* ranks, int max_als_sweeps) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (!h->canonical) throw std::invalid_argument("no canonical sum built");
    TruncationSpec spec;
    if (eps > 0.0) spec.tolerance = eps;
    if (ranks) spec.ranks = Dims3{ranks[0], ranks[1], ranks[2]};
    if (max_als_sweeps >= 0) spec.max_als_sweeps = max_als_sweeps;
    auto [t, rep] = mode == 0 ? rhosvd(*h->canonical, spec) : canonical_to_tucker(*h->canonical, spec);
    h->tucker = std::move(t);
    h->report = std::move(rep);
  });
}

// ranks[3]; n_sv[3]; rep = {bound_abs, bound_rel, weight_norm, input_norm, stability_constant,
// stability_ok}; ties[3]
int lref_tucker_info(void* hp, int64_t* ranks, int64_t* n_sv, double* rep, int* ties) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (!h->tucker) throw std::invalid_argument("no reduction run");
    const Dims3 r = h->tucker->ranks();
    for (int l = 0; l < 3; ++l) {
      ranks[l] = r[l];
      n_sv[l] = h->report->singular_values[l].size();
      ties[l] = h->report->tie_at_cutoff[l] ? 1 : 0;
    }
    rep[0] = h->report->bound_abs;
    rep[1] = h->report->bound_rel;
    rep[2] = h->report->weight_norm;
    rep[3] = h->report->input_norm;
    rep[4] = h->report->stability_constant;
    rep[5] = h->report->stability_ok ? 1.0 : 0.0;
  });
}

int lref_tucker_copy(void* hp, double* core, double* u0, double* u1, double* u2, double* sv0,
                     double* sv1, double* sv2) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (!h->tucker) throw std::invalid_argument("no reduction run");
    if (core)
      std::memcpy(core, h->tucker->core().data().data(), sizeof(double) * size_t(h->tucker->core().size()));
    double* u[3] = {u0, u1, u2};
    double* sv[3] = {sv0, sv1, sv2};
    for (int l = 0; l < 3; ++l) {
      copy_matrix(h->tucker->factor(l), u[l]);
      if (sv[l])
        std::memcpy(sv[l], h->report->singular_values[l].data(),
                    sizeof(double) * size_t(h->report->singular_values[l].size()));
    }
  });
}

// which: 0 canonical sum entries, 1 Tucker entries, 2 brute-force oracle_entry over all sources
int lref_entries(void* hp, int which, int64_t n, const int64_t* probes, double* out) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    for (int64_t p = 0; p < n; ++p) {
      const Index i = probes[3 * p], j = probes[3 * p + 1], k = probes[3 * p + 2];
      if (which == 0) {
        if (!h->canonical) throw std::invalid_argument("no canonical sum built");
        out[p] = h->canonical->entry(i, j, k);
      } else if (which == 1) {
        if (!h->tucker) throw std::invalid_argument("no reduction run");
        out[p] = h->tucker->entry(i, j, k);
      } else {
        out[p] = oracle_entry<double>(h->sources, h->refs, i, j, k);
      }
    }
  });
}

static int64_t emit(const std::string& text, char* buf, int64_t cap) {
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(text.size(), size_t(cap - 1));
    std::memcpy(buf, text.data(), n);
    buf[n] = 0;
  }
  return int64_t(text.size());
}

// write_spectral_report (src/report.cpp:28-47) of the last reduction; returns the text length
int64_t lref_spectral_report_text(void* hp, char* buf, int64_t cap) {
  Handle* h = static_cast<Handle*>(hp);
  int64_t n = -1;
  guarded(h, [&] {
    if (!h->report) throw std::invalid_argument("no reduction run");
    std::ostringstream os;
    write_spectral_report(os, *h->report);
    n = emit(os.str(), buf, cap);
  });
  return n;
}

// write_provenance (src/report.cpp:49-73) of the sum as cmd_sum records it (commands.cpp:56-72):
// reduced != 0: the Tucker result with its report, else the canonical sum
int64_t lref_provenance_text(void* hp, uint64_t seed, int reduced, const char* extra, char* buf,
                             int64_t cap) {
  Handle* h = static_cast<Handle*>(hp);
  int64_t n = -1;
  guarded(h, [&] {
    if (!h->canonical) throw std::invalid_argument("no canonical sum built");
    LatticeSumResult<double> res;
    res.geometry = h->out_geometry;
    res.grid = h->ref.base_grid;
    res.provenance = h->provenance;
    if (reduced) {
      if (!h->tucker) throw std::invalid_argument("no reduction run");
      res.tensor = *h->tucker;
      res.report = *h->report;
    } else {
      res.tensor = *h->canonical;
    }
    std::vector<std::string> lines;
    if (extra && *extra) lines.push_back(extra);
    std::ostringstream os;
    write_provenance(os, res, seed, lines);
    n = emit(os.str(), buf, cap);
  });
  return n;
}

// write_tensor (src/tensor_io.cpp): which 0 = the canonical sum, 1 = the Tucker result
int lref_write_tensor(void* hp, int which, const char* path) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    if (which == 0) {
      if (!h->canonical) throw std::invalid_argument("no canonical sum built");
      write_tensor(path, TensorVariant(*h->canonical));
    } else {
      if (!h->tucker) throw std::invalid_argument("no reduction run");
      write_tensor(path, TensorVariant(*h->tucker));
    }
  });
}

// read_tensor (src/tensor_io.cpp) + entries of what was read; kind_out: 0 canonical, 1 Tucker;
// returns 5 on a TensorIoError (bad magic / version / checksum / truncation)
int lref_read_tensor_entries(const char* path, int* kind_out, int64_t* dims, int64_t n,
                             const int64_t* probes, double* out) {
  try {
    const TensorVariant t = read_tensor(path);
    const bool can = std::holds_alternative<CanonicalTensor<double>>(t);
    if (kind_out) *kind_out = can ? 0 : 1;
    const Dims3 d = can ? std::get<CanonicalTensor<double>>(t).dims() : std::get<TuckerTensor<double>>(t).dims();
    for (int l = 0; l < 3; ++l) dims[l] = d[l];
    for (int64_t p = 0; p < n; ++p) {
      const Index i = probes[3 * p], j = probes[3 * p + 1], k = probes[3 * p + 2];
      out[p] = can ? std::get<CanonicalTensor<double>>(t).entry(i, j, k)
                   : std::get<TuckerTensor<double>>(t).entry(i, j, k);
    }
    return 0;
  } catch (const TensorIoError& e) {
    g_error = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 9;
  }
}

static RunConfig run_config(const Handle* h, uint64_t seed) {
  RunConfig cfg;
  cfg.kernel = h->geom.kernel;
  cfg.n = h->n_per_cell;
  cfg.b = h->geom.cell_width;
  cfg.quad_M = h->M;
  cfg.geometry = h->canonical || h->tucker ? h->out_geometry : h->geom;
  cfg.has_geometry = true;
  cfg.sublattices = h->placements;
  cfg.seed = seed;
  return cfg;
}

// cmd_sum (src/commands.cpp:108-177), the caller of the hot path: the geometry given to
// lref_create plus the defect clusters (as in lref_sum) or sublattices, optional truncation
// eps > 0 (canonical_to_tucker), writing the tensor / provenance / report files whose paths are
// non-empty.  The result stays in the handle (canonical sum, or Tucker result + report).
int lref_cmd_sum(void* hp, int n_sub, const int* sub_cells, const double* sub_offsets, int n_def,
                 const int* def_nsites, const int* def_sites, const double* def_charge,
                 const double* def_goff, const int* def_kind, double eps, int max_als_sweeps,
                 uint64_t seed, const char* tensor_path, const char* provenance_path,
                 const char* report_path, char* logbuf, int64_t cap) {
  Handle* h = static_cast<Handle*>(hp);
  return guarded(h, [&] {
    h->canonical.reset();
    h->tucker.reset();
    h->report.reset();
    h->placements.clear();
    RunConfig cfg = run_config(h, seed);
    cfg.geometry.defects.clear();
    for (int s = 0; s < n_sub; ++s) {
      SublatticePlacement p;
      p.geom = h->geom;
      p.geom.active = {};
      p.geom.cells = {sub_cells[3 * s], sub_cells[3 * s + 1], sub_cells[3 * s + 2]};
      p.offset_cells = Array3<double>(sub_offsets[3 * s], sub_offsets[3 * s + 1], sub_offsets[3 * s + 2]);
      cfg.sublattices.push_back(std::move(p));
    }
    const int* site = def_sites;
    for (int d = 0; d < n_def; ++d) {
      DefectSpec spec;
      for (int s = 0; s < def_nsites[d]; ++s, site += 3) spec.sites.push_back({site[0], site[1], site[2]});
      spec.kind = def_kind && def_kind[d] ? DefectKind::impurity : DefectKind::vacancy;
      spec.charge = def_charge[d];
      if (def_goff)
        spec.grid_offset = Array3<double>(def_goff[3 * d], def_goff[3 * d + 1], def_goff[3 * d + 2]);
      cfg.geometry.defects.push_back(std::move(spec));
    }
    if (eps > 0.0) {
      cfg.truncation = TruncationSpec::tol(eps);
      if (max_als_sweeps >= 0) cfg.truncation->max_als_sweeps = max_als_sweeps;
    }
    if (tensor_path) cfg.output_tensor = tensor_path;
    if (provenance_path) cfg.output_provenance = provenance_path;
    if (report_path) cfg.output_report = report_path;
    std::ostringstream log;
    LatticeSumResult<double> res = cmd_sum(cfg, log);
    emit(log.str(), logbuf, cap);
    h->placements = cfg.sublattices;
    h->out_geometry = res.geometry;
    if (n_sub == 0) h->out_geometry.defects = cfg.geometry.defects;
    h->provenance = res.provenance;
    if (res.is_canonical()) {
      h->canonical = res.canonical();
    } else {
      h->tucker = res.tucker_tensor();
      h->report = res.report;
    }
  });
}

// cmd_verify (src/commands.cpp:200-284) of a stored tensor file against the brute-force oracle of
// the handle's geometry (as last summed): `probes` mt19937_64(seed) probes, gated by bound_abs
// (>= 0), else the provenance file's recorded bound, else `tolerance`.  0: "verify: ok";
// 6: VerificationError; 5: TensorIoError.  The reference's log text goes to logbuf.
int lref_cmd_verify(void* hp, const char* tensor_path, const char* provenance_path, int probes,
                    double tolerance, double bound_abs, uint64_t seed, char* logbuf, int64_t cap) {
  Handle* h = static_cast<Handle*>(hp);
  std::ostringstream log;
  int rc = 0;
  try {
    const RunConfig cfg = run_config(h, seed);
    VerifyOptions vo;
    vo.tensor_path = tensor_path;
    if (provenance_path) vo.provenance_path = provenance_path;
    vo.probes = probes;
    vo.tolerance = tolerance;
    vo.bound_abs = bound_abs;
    cmd_verify(cfg, vo, log);
  } catch (const VerificationError& e) {
    h->error = e.what();
    rc = 6;
  } catch (const TensorIoError& e) {
    h->error = e.what();
    rc = 5;
  } catch (const std::exception& e) {
    h->error = e.what();
    rc = 9;
  }
  emit(log.str(), logbuf, cap);
  return rc;
}

// detail::assembled_vector on one reference column with explicit K set, n, offset (lattice_sum.hpp:101-144)
int lref_assembled_vector(const double* ref, int64_t ref_len, const int* kset, int nk, int64_t n,
                          long off, int64_t nl, int accumulation, double* out) {
  return guarded(nullptr, [&] {
    VectorX<double> r(ref_len);
    std::memcpy(r.data(), ref, sizeof(double) * size_t(ref_len));
    const Accumulation acc = accumulation == 0   ? Accumulation::sliding
                             : accumulation == 1 ? Accumulation::ascending
                                                 : Accumulation::compensated;
    const VectorX<double> v =
        detail::assembled_vector<double>(r, std::span<const int>(kset, size_t(nk)), n, off, nl, acc, 0);
    std::memcpy(out, v.data(), sizeof(double) * size_t(nl));
  });
}

// detail::rank_for_tolerance (rank_reduction.hpp:73-84)
int64_t lref_rank_for_tolerance(const double* sv, int64_t n, double eps) {
  VectorX<double> v(n);
  std::memcpy(v.data(), sv, sizeof(double) * size_t(n));
  return detail::rank_for_tolerance(v, eps);
}

// default_step_constant (quadrature.hpp:238-269) and build_quadrature (quadrature.hpp:124-187) on shell [a, A]
int lref_quadrature(int family, double lam, int M, double C0, double a, double A, double* c0_out,
                    double* nodes, double* weights) {
  return guarded(nullptr, [&] {
    const KernelSpec k = make_kernel(family, lam);
    const auto& term = k.terms().at(0);
    const Shell shell{a, A};
    const double c0 = C0 > 0.0 ? C0 : default_step_constant(term.primitive, M, shell);
    if (c0_out) *c0_out = c0;
    const auto rule = build_quadrature<double>(term.primitive, M, c0, shell);
    if (nodes) std::memcpy(nodes, rule.nodes.data(), sizeof(double) * size_t(rule.size()));
    if (weights) std::memcpy(weights, rule.weights.data(), sizeof(double) * size_t(rule.size()));
  });
}

}  // extern "C"
