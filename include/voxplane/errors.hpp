// Reference-compatible include path (voxplane/errors.hpp): the B200 API lives in
// voxplane/voxplane.hpp.
#pragma once
#include "voxplane/voxplane.hpp"
