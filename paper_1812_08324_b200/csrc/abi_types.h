// Definitions of the opaque handle types of include/levyh_b200.h (shared by the library and
// the testing library, csrc/testing/).
#pragma once

#include <memory>

#include "core.h"

struct lh_ctx {
    lh::Ctx c;
};
struct lh_tree {
    std::shared_ptr<lh::Tree> t;
};
struct lh_hmat {
    lh::HMat h;
};
