// TEST INFRASTRUCTURE (oracle/): the reference's on-disk reference-tensor cache
// (/root/reference/proj/src/cache.cpp) needs nlohmann json, which is absent, and the cache is out
// of scope.  These three definitions satisfy include/latsum/cache.hpp:12-27 with
// "never cached", so that the reference's own src/commands.cpp (cmd_sum, cmd_verify, cmd_bench)
// links into oracle/_ref unchanged: every reference is built by build_reference_canonical.
#include "latsum/cache.hpp"

namespace latsum {

std::string resolve_cache_dir(const std::optional<std::string>& config_override) {
  return config_override ? *config_override : std::string("latsum_cache");
}

std::optional<ReferenceTensor<double>> try_load_reference(const std::string&, const KernelSpec&,
                                                          const UniformGrid<double>&, int, double,
                                                          bool) {
  return std::nullopt;
}

void store_reference(const std::string&, const ReferenceTensor<double>&, double) {}

}  // namespace latsum
