// C++ drop-in check: the reference's own unit-test scenarios written against
// include/latsum_b200/latsum.hpp (reference names, exception types), run on the GPU.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "latsum_b200/latsum.hpp"

using namespace latsum;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

int main() {
  // reference side matrices: 2n rows, R = 2M+1, unit columns (test_reference.cpp:49-60)
  auto grid = UniformGrid::cubic(4.0, 32);
  auto ref = build_reference_canonical(KernelSpec::newton(), grid, 10);
  CHECK(ref.rank() == 21);
  const auto f = ref.factor(0);
  CHECK(f.size() == size_t(64 * 21));
  double nrm = 0;
  for (int i = 0; i < 64; ++i) nrm += f[i] * f[i];
  CHECK(std::abs(nrm - 1.0) < 1e-14);

  // odd cell counts are rejected (test_grid_geometry.cpp:20-26)
  try {
    build_reference_canonical(KernelSpec::newton(), UniformGrid::cubic(1.0, 7), 4);
    CHECK(false);
  } catch (const std::invalid_argument&) {
  }

  // single vacancy: rank 2R and entry = base - window (test_lattice_sum.cpp:198-232)
  LatticeGeometry geom;
  geom.cells = {4, 4, 4};
  const Index n = 16;
  auto ref2 = build_reference_canonical(KernelSpec::newton(), lattice_grid(geom, n), 8);
  auto base = assembled_sum_canonical(ref2, geom, n);
  CHECK(base.rank() == ref2.rank());
  LatticeGeometry vg = geom;
  DefectSpec vac;
  vac.sites = {{0, 0, 0}};
  vac.charge = -1.0;
  vg.defects = {vac};
  auto defected = defected_sum(ref2, vg, n);
  CHECK(defected.rank() == 2 * ref2.rank());
  double worst = 0, scale = 0;
  for (int p = 0; p < 50; ++p) {
    const Index i = (7 * p) % 64, j = (13 * p + 5) % 64, k = (29 * p + 3) % 64;
    const double d = defected.entry(i, j, k), b = base.entry(i, j, k);
    worst = std::fmax(worst, std::abs(b - d));
    scale = std::fmax(scale, std::abs(b));
  }
  CHECK(worst > 0 && worst < scale);  // the vacancy removes a positive window

  // window overflow names the mode (grid.hpp:87-114)
  LatticeGeometry og = geom;
  DefectSpec far;
  far.sites = {{0, 9, 0}};
  far.kind = DefectKind::impurity;
  far.charge = 1.0;
  og.defects = {far};
  try {
    defected_sum(ref2, og, n);
    CHECK(false);
  } catch (const WindowOverflowError& e) {
    CHECK(e.mode() == 2);
  }

  // rhosvd: fixed ranks reproduce an exact low-rank input (test_rank_reduction.cpp:22-41)
  LatticeGeometry small;
  small.cells = {2, 2, 2};
  auto ref3 = build_reference_canonical(KernelSpec::newton(), lattice_grid(small, 8), 3);
  auto can = assembled_sum_canonical(ref3, small, 8);
  auto [t, rep] = rhosvd(can, TruncationSpec::fixed_ranks(10, 10, 10));
  for (int l = 0; l < 3; ++l) CHECK(rep.chosen_ranks[l] <= 7);
  const auto dense = to_dense(t);
  double err = 0, mx = 0;
  for (Index k = 0; k < 16; ++k)
    for (Index j = 0; j < 16; ++j)
      for (Index i = 0; i < 16; ++i) {
        const double c = can.entry(i, j, k);
        err = std::fmax(err, std::abs(dense[i + 16 * (j + 16 * k)] - c));
        mx = std::fmax(mx, std::abs(c));
      }
  CHECK(err <= 1e-12 * mx);
  CHECK(rep.input_norm > 0 && rep.weight_norm > 0);

  // tolerance-driven truncation stays within the bound
  auto [t2, rep2] = rhosvd(defected, TruncationSpec::tol(1e-6));
  CHECK(t2.ranks()[0] >= 1 && t2.ranks()[0] <= 64);
  CHECK(rep2.bound_abs >= 0.0);

  try {
    rhosvd(can, TruncationSpec{});
    CHECK(false);
  } catch (const std::invalid_argument&) {
  }
  // the reference's result-level interface: rectangular clusters assemble at reference
  // rank, ragged ones per site (test_lattice_sum.cpp:273-305)
  {
    LatticeGeometry g8;
    g8.cells = {8, 8, 1};
    const Index n8 = 8;
    ReferenceSet refs;
    refs.add(build_reference_canonical(KernelSpec::newton(), lattice_grid(g8, n8), 8));
    const ReferenceTensor& r8 = refs.find(KernelSpec::newton());
    const Index R = r8.rank();
    LatticeSumResult base8 = assembled_sum_result(r8, g8);
    CHECK(base8.canonical().rank() == R);
    DefectSpec cluster;
    cluster.kind = DefectKind::vacancy;
    cluster.sites = {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}, {1, 1, 0}};
    cluster.charge = -1.0;
    auto out = defected_sum(base8, {cluster}, refs, std::nullopt);
    CHECK(out.canonical().rank() == 2 * R);
    DefectSpec ragged;
    ragged.kind = DefectKind::vacancy;
    ragged.sites = {{2, 2, 0}, {2, 3, 0}, {3, 2, 0}};
    ragged.charge = -1.0;
    auto out2 = defected_sum(base8, {ragged}, refs, std::nullopt);
    CHECK(out2.canonical().rank() == (1 + 3) * R);
    auto both = defected_sum(base8, {cluster, ragged}, refs, std::nullopt);
    CHECK(both.canonical().rank() == (1 + 1 + 3) * R);
    CHECK(both.provenance.size() == 3 && both.provenance[1].canonical_rank == R &&
          both.provenance[2].canonical_rank == 3 * R && both.provenance[2].sites == 3);
    // sequential == joint (test_lattice_sum.cpp:248-270)
    auto seq = defected_sum(defected_sum(base8, {cluster}, refs, std::nullopt), {ragged}, refs,
                            std::nullopt);
    double worst = 0, scale = 0;
    for (int p = 0; p < 40; ++p) {
      const Index i = (11 * p) % 64, j = (17 * p + 3) % 64, k = (5 * p) % 8;
      worst = std::fmax(worst, std::abs(seq.canonical().entry(i, j, k) - both.canonical().entry(i, j, k)));
      scale = std::fmax(scale, std::abs(both.canonical().entry(i, j, k)));
    }
    CHECK(worst <= 1e-13 * scale);
    // truncated: canonical_to_tucker, report and provenance sidecar (report.cpp:28-73)
    auto tr = defected_sum(base8, {cluster, ragged}, refs, TruncationSpec::tol(1e-6));
    CHECK(!tr.is_canonical() && tr.report.has_value());
    std::ostringstream rs, ps;
    write_spectral_report(rs, *tr.report);
    write_provenance(ps, tr, 42);
    CHECK(rs.str().rfind("# spectral report\nchosen_ranks ", 0) == 0);
    CHECK(ps.str().find("format tucker\n") != std::string::npos);
    CHECK(ps.str().find("summand \"vacancy cluster\" rank " + std::to_string(R) + " sites 4\n") !=
          std::string::npos);
    CHECK(ps.str().find("truncation_bound_abs ") != std::string::npos);
    // a defect with its own kernel (DefectSpec.kernel, lattice_sum.hpp:301-303) needs that
    // kernel's reference tensor in the set ...
    DefectSpec yk = ragged;
    yk.kind = DefectKind::impurity;
    yk.charge = 0.5;
    yk.kernel = KernelSpec::yukawa(0.5);
    try {
      defected_sum(base8, {yk}, refs, std::nullopt);
      CHECK(false);
    } catch (const std::invalid_argument&) {  // no reference built for it
    }
    // ... and is then summed in DefectSpec order by add_concat (lattice_sum.hpp:372-374):
    // rank, provenance, and entries = the Newton sum + the Yukawa windows alone
    refs.add(build_reference_canonical(KernelSpec::yukawa(0.5), lattice_grid(g8, n8), 8));
    const ReferenceTensor& ry = refs.find(KernelSpec::yukawa(0.5));
    auto mixed = defected_sum(base8, {cluster, yk, ragged}, refs, std::nullopt);
    CHECK(mixed.canonical().rank() == (1 + 1) * R + 3 * ry.rank() + 3 * R);
    CHECK(mixed.provenance.size() == 4 && mixed.provenance[2].label == "impurity cluster" &&
          mixed.provenance[2].canonical_rank == 3 * ry.rank());
    LatticeGeometry only_yk;  // the Yukawa cluster alone: windows of the Yukawa reference
    only_yk.cells = g8.cells;
    detail::Blocks by;
    detail::add_defect(by, yk, n8);
    auto yk_alone = assemble(ry, by);
    worst = 0;
    scale = 0;
    for (int p = 0; p < 40; ++p) {
      const Index i = (11 * p) % 64, j = (17 * p + 3) % 64, k = (5 * p) % 8;
      const double want = both.canonical().entry(i, j, k) + yk_alone.entry(i, j, k);
      worst = std::fmax(worst, std::abs(mixed.canonical().entry(i, j, k) - want));
      scale = std::fmax(scale, std::abs(want));
    }
    CHECK(worst <= 1e-13 * scale);
    // a result of mixed kernels can be extended and truncated like any other
    auto mixed2 = defected_sum(mixed, {cluster}, refs, TruncationSpec::tol(1e-6));
    CHECK(!mixed2.is_canonical() && mixed2.provenance.size() == 5);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
