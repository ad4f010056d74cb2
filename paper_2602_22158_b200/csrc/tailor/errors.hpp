// Error taxonomy of the tailoring path. The kinds, their printed names and the
// user-vs-internal split are the reference's contract
// (R/include/tailor/errors.hpp:12-62): user errors map to CLI exit 1,
// Consistency / NonFinite / Storage to exit 2. Across the C ABI the kind
// travels as an int code (include/tailor_b200.h, TG_E_*); no exception ever
// crosses it.
#pragma once

#include <stdexcept>
#include <string>

namespace tailor {

enum class ErrorKind : int {
    InvalidModule = 1,
    Geometry,
    NonFinite,
    Recipe,
    SourceLacksModule,
    MissingArtifact,
    CorruptContainer,
    UnrecoverableModule,
    MissingModules,
    Consistency,
    Storage,
    Device,  // CUDA failure; reported as a Storage-class (exit 2) error
};

const char* error_kind_name(ErrorKind kind);

class TailorError : public std::runtime_error {
  public:
    TailorError(ErrorKind kind, const std::string& message)
        : std::runtime_error(std::string(error_kind_name(kind)) + ": " + message), kind_(kind) {}
    ErrorKind kind() const { return kind_; }
    bool is_user_error() const {
        return kind_ != ErrorKind::Consistency && kind_ != ErrorKind::NonFinite &&
               kind_ != ErrorKind::Storage && kind_ != ErrorKind::Device;
    }

  private:
    ErrorKind kind_;
};

[[noreturn]] void fail(ErrorKind kind, const std::string& message);

} // namespace tailor
