// Text reports of the lattice-sum path (host only): the spectral report and the provenance
// sidecar that `latsum sum` writes next to the tensor file (report.cpp:28-73,
// commands.cpp:56-72).  Same text, byte for byte: 17 significant digits in the stream's
// default float format (report.cpp:9-12), so reruns diff byte-identically.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "latsum_b200.h"

namespace {

// std::ostream with precision(17) and no floatfield prints doubles as printf's %.17g
void put_double(std::string& s, double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  s += b;
}

void put_int(std::string& s, int64_t v) {
  char b[24];
  std::snprintf(b, sizeof b, "%" PRId64, v);
  s += b;
}

int64_t emit(const std::string& s, char* buf, int64_t cap) {
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(s.size(), size_t(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return int64_t(s.size());
}

}  // namespace

extern "C" {

int64_t latsum_format_spectral_report(const latsum_spectral_report* r, const double* const sigma[3],
                                      char* buf, int64_t cap) {
  if (!r) return -1;
  std::string s = "# spectral report\n";
  s += "chosen_ranks ";
  put_int(s, r->chosen_ranks[0]);
  s += " ";
  put_int(s, r->chosen_ranks[1]);
  s += " ";
  put_int(s, r->chosen_ranks[2]);
  s += "\nbound_abs ";
  put_double(s, r->bound_abs);
  s += "\nbound_rel ";
  put_double(s, r->bound_rel);
  s += "\nweight_norm ";
  put_double(s, r->weight_norm);
  s += "\ninput_norm ";
  put_double(s, r->input_norm);
  s += "\nstability_constant ";
  put_double(s, r->stability_constant);
  s += "\nstability_ok ";
  s += r->stability_ok ? "1" : "0";
  s += "\n";
  for (int l = 0; l < 3; ++l) {
    s += "sigma_mode";
    put_int(s, l + 1);
    if (r->tie_at_cutoff[l]) s += " (tie at cutoff)";
    if (sigma && sigma[l])
      for (int64_t k = 0; k < r->n_singular[l]; ++k) {
        s += " ";
        put_double(s, sigma[l][k]);
      }
    s += "\n";
  }
  return emit(s, buf, cap);
}

int64_t latsum_format_provenance(const latsum_provenance* p, char* buf, int64_t cap) {
  if (!p) return -1;
  std::string s = "# lattice sum provenance\nseed ";
  char b[24];
  std::snprintf(b, sizeof b, "%" PRIu64, p->seed);
  s += b;
  s += "\ngrid ";
  for (int l = 0; l < 3; ++l) {
    if (l) s += " ";
    put_int(s, p->grid[l]);
  }
  s += "\ncells ";
  for (int l = 0; l < 3; ++l) {
    if (l) s += " ";
    put_int(s, p->cells[l]);
  }
  if (p->format == 0) {
    s += "\nformat canonical\nrank ";
    put_int(s, p->rank);
  } else {
    s += "\nformat tucker\nranks ";
    for (int l = 0; l < 3; ++l) {
      if (l) s += " ";
      put_int(s, p->ranks[l]);
    }
  }
  s += "\nsummands ";
  put_int(s, p->nsummands);
  s += "\n";
  for (int64_t i = 0; i < p->nsummands; ++i) {
    s += "summand \"";
    s += p->labels && p->labels[i] ? p->labels[i] : "";
    s += "\" rank ";
    put_int(s, p->summand_ranks ? p->summand_ranks[i] : 0);
    s += " sites ";
    put_int(s, p->summand_sites ? p->summand_sites[i] : 0);
    s += "\n";
  }
  if (p->has_report) {
    s += "truncation_bound_abs ";
    put_double(s, p->bound_abs);
    s += "\ntruncation_bound_rel ";
    put_double(s, p->bound_rel);
    s += "\n";
  }
  for (int64_t i = 0; i < p->nextra; ++i) {
    s += p->extra && p->extra[i] ? p->extra[i] : "";
    s += "\n";
  }
  return emit(s, buf, cap);
}

}  // extern "C"
