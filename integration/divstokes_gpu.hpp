// Reference-side drop-in: the one header a divstokes maintainer includes to
// route solve_stokes onto the B200 solver (include/dsgpu.h). See INTEGRATION.md.
#pragma once

#include <string>

#include "divstokes/precond.hpp"

namespace divstokes_gpu {

// Same contract as divstokes::solve_stokes(system, strategy, options)
// (proj/include/divstokes/precond.hpp:68-69): the preconditioner setup is
// the reference's own (rcm_permutation -> permute_symmetric -> ic0, as
// PcgBlock does, proj/src/precond.cpp:61-64), the MINRES loop runs on the
// GPU, the zero-mean pressure filter is the reference's (precond.cpp:266-284).
// Strategies: PCG(A,Q), PCG(A)+Diag(Q), Diag(A,Q), IC0-PCG(A,Q),
// IC0-PCG(A)+Diag(Q). Throws the reference's exception types.
divstokes::StokesSolution solve_stokes(const divstokes::StokesSystem& system,
                                       const std::string& strategy,
                                       const divstokes::SolverOptions& options, int device = 0);

}  // namespace divstokes_gpu
