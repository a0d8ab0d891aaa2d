#include "core.h"
namespace lh {
void hlu(Ctx &, HMat &, double) { throw Error(LH_EINTERNAL, "hlu not built yet"); }
void solve(Ctx &, HMat &, double *, i64, int, int) { throw Error(LH_EINTERNAL, "solve not built yet"); }
void prepare_inverse(Ctx &, HMat &, double) { throw Error(LH_EINTERNAL, "not built yet"); }
void cn_steps(Ctx &, HMat &, HMat &, double *, i64, int, int, int) { throw Error(LH_EINTERNAL, "not built yet"); }
}
