// Host-side core of the B200 drop-in: the reference's error taxonomy
// (reference proj/include/vpinn/core.hpp:17-114) and its splitmix64 stream
// (core.hpp:119-154), which seeds weight init and point sampling bit-exactly.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace vpinn {

// ErrorCategory values double as CLI exit codes and C-ABI return codes.
enum class ErrorCategory : int { config = 2, mesh = 3, numeric = 4, io = 5, device = 6 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCategory c, const std::string& m) : std::runtime_error(m), cat_(c) {}
  ErrorCategory category() const noexcept { return cat_; }
  int code() const noexcept { return static_cast<int>(cat_); }

 private:
  ErrorCategory cat_;
};

#define VPINN_ERROR_TYPE(Name, Cat)                                                \
  struct Name : Error {                                                            \
    explicit Name(const std::string& m) : Error(ErrorCategory::Cat, m) {}          \
  };
VPINN_ERROR_TYPE(InvalidArgumentError, config)
VPINN_ERROR_TYPE(ConfigError, config)
VPINN_ERROR_TYPE(InvalidModeError, config)
VPINN_ERROR_TYPE(MeshFileError, mesh)
VPINN_ERROR_TYPE(AssemblyError, numeric)
VPINN_ERROR_TYPE(NumericOverflowError, numeric)
VPINN_ERROR_TYPE(ContractViolationError, numeric)
VPINN_ERROR_TYPE(IoError, io)
VPINN_ERROR_TYPE(DeviceError, device)
#undef VPINN_ERROR_TYPE

struct DegenerateElementError : Error {
  DegenerateElementError(int id, const std::string& m) : Error(ErrorCategory::mesh, m), id_(id) {}
  int element_id() const noexcept { return id_; }
  int id_;
};

struct TrainingAbortError : Error {
  TrainingAbortError(std::int64_t step, const std::string& m)
      : Error(ErrorCategory::numeric, m), step_(step) {}
  std::int64_t step() const noexcept { return step_; }
  std::int64_t step_;
};

// Seeded generator used wherever a seed appears in an interface.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : x_(seed) {
    (void)bits();
    (void)bits();
  }
  std::uint64_t bits() {
    x_ += 0x9e3779b97f4a7c15ull;
    std::uint64_t z = x_;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  std::uint64_t integer(std::uint64_t n) {
    return static_cast<std::uint64_t>(uniform() * static_cast<double>(n));
  }

 private:
  std::uint64_t x_;
};

}  // namespace vpinn
