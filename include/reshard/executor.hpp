// Reference header name (proj/include/reshard/executor.hpp) forwarded to the
// B200 implementation, so reference callers compile unchanged.
#pragma once
#include "reshard_b200/reshard.hpp"
