// ginsim/errors.hpp — C++ error types of the B200 GIN host API.
//
// Same names and hierarchy as the reference (proj/core/include/ginsim/
// errors.hpp:10-52) so callers catch precisely; each maps one-to-one onto a
// ginsim_status code of the C ABI (include/ginsim_cuda.h), and throw_status()
// turns a failed C call back into the typed exception.
#pragma once

#include <stdexcept>
#include <string>

#include "../ginsim_cuda.h"

namespace ginsim {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

#define GINSIM_B200_ERROR(Name)  \
  class Name : public Error {    \
   public:                       \
    using Error::Error;          \
  }

GINSIM_B200_ERROR(InvalidDescriptor);
GINSIM_B200_ERROR(MalformedDescriptor);
GINSIM_B200_ERROR(OutOfBounds);
GINSIM_B200_ERROR(UnknownWindow);
GINSIM_B200_ERROR(RankOutOfRange);
GINSIM_B200_ERROR(DuplicateEndpoint);
GINSIM_B200_ERROR(UnknownChannel);
GINSIM_B200_ERROR(MalformedFrame);
GINSIM_B200_ERROR(UnknownHandle);
GINSIM_B200_ERROR(BackendMismatch);
GINSIM_B200_ERROR(InvalidContext);
GINSIM_B200_ERROR(ConfigMismatch);
GINSIM_B200_ERROR(BootstrapTimeout);
GINSIM_B200_ERROR(RegistrationMismatch);
GINSIM_B200_ERROR(InvalidPeer);
GINSIM_B200_ERROR(InvalidSignal);
GINSIM_B200_ERROR(InvalidCounter);
GINSIM_B200_ERROR(ResetWhileOutstanding);
GINSIM_B200_ERROR(Timeout);
GINSIM_B200_ERROR(VerificationFailure);
GINSIM_B200_ERROR(FlowControlViolation);
GINSIM_B200_ERROR(ChildFailure);
GINSIM_B200_ERROR(UsageError);
GINSIM_B200_ERROR(CudaError);

#undef GINSIM_B200_ERROR

[[noreturn]] inline void throw_status(int code, const std::string& what) {
  switch (code) {
    case GINSIM_E_INVALID_DESCRIPTOR: throw InvalidDescriptor(what);
    case GINSIM_E_MALFORMED_DESCRIPTOR: throw MalformedDescriptor(what);
    case GINSIM_E_OUT_OF_BOUNDS: throw OutOfBounds(what);
    case GINSIM_E_UNKNOWN_WINDOW: throw UnknownWindow(what);
    case GINSIM_E_RANK_OUT_OF_RANGE: throw RankOutOfRange(what);
    case GINSIM_E_DUPLICATE_ENDPOINT: throw DuplicateEndpoint(what);
    case GINSIM_E_UNKNOWN_CHANNEL: throw UnknownChannel(what);
    case GINSIM_E_MALFORMED_FRAME: throw MalformedFrame(what);
    case GINSIM_E_UNKNOWN_HANDLE: throw UnknownHandle(what);
    case GINSIM_E_BACKEND_MISMATCH: throw BackendMismatch(what);
    case GINSIM_E_INVALID_CONTEXT: throw InvalidContext(what);
    case GINSIM_E_CONFIG_MISMATCH: throw ConfigMismatch(what);
    case GINSIM_E_BOOTSTRAP_TIMEOUT: throw BootstrapTimeout(what);
    case GINSIM_E_REGISTRATION_MISMATCH: throw RegistrationMismatch(what);
    case GINSIM_E_INVALID_PEER: throw InvalidPeer(what);
    case GINSIM_E_INVALID_SIGNAL: throw InvalidSignal(what);
    case GINSIM_E_INVALID_COUNTER: throw InvalidCounter(what);
    case GINSIM_E_RESET_WHILE_OUTSTANDING: throw ResetWhileOutstanding(what);
    case GINSIM_E_TIMEOUT: throw Timeout(what);
    case GINSIM_E_VERIFICATION_FAILURE: throw VerificationFailure(what);
    case GINSIM_E_FLOW_CONTROL_VIOLATION: throw FlowControlViolation(what);
    case GINSIM_E_CHILD_FAILURE: throw ChildFailure(what);
    case GINSIM_E_USAGE: throw UsageError(what);
    case GINSIM_E_CUDA: throw CudaError(what);
    default: throw Error(what);
  }
}

// Checks a C-ABI status and rethrows it as the matching typed exception.
inline void check(int status) {
  if (status != GINSIM_OK) throw_status(status, ginsim_cuda_last_error());
}

}  // namespace ginsim
