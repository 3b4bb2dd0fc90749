// Reference-side adapter API: irkprec's irk_step /
// integrate signatures (irk.hpp:36-39, 54-58) solved on the B200 through the
// C ABI of include/irkdev.h.  A maintainer adds this header and
// irk_step_b200.cpp to irkprec; the overloads without B200Options keep the
// reference's exact signatures and semantics (full GMRES, default AmgParams).
#ifndef IRK_B200_HPP
#define IRK_B200_HPP

#include <span>

#include "irkprec/amg.hpp"
#include "irkprec/butcher.hpp"
#include "irkprec/gmres.hpp"
#include "irkprec/irk.hpp"
#include "irkprec/stage.hpp"

namespace irkprec {

// Device-side options the reference's GmresConfig / BlockPreconditioner do
// not carry.  restart = 0 is full GMRES -- the reference's gmres.hpp:20
// behaviour, and the default; restart = m > 0 runs GMRES(m) (BASELINE's
// GMRES(50)).  `amg` must be the AmgParams the BlockPreconditioner was built
// with (BlockPreconditioner keeps them private, stage.hpp:92); the adapter
// checks the device hierarchies against P->hierarchy_stats() and refuses a
// mismatch instead of silently solving with another hierarchy.
struct B200Options {
    int restart = 0;
    AmgParams amg{};
    int device = 0;
};

IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg);
IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg, const B200Options& opt);
TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg);
TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg,
                                 const B200Options& opt);
/// Frees the calling thread's cached device solvers (irk_step_b200 keeps up
/// to IRK_B200_CACHE of them, default 4, keyed on content).
void irk_b200_release();

}  // namespace irkprec

#endif
