"""B200-native sequence criteria (wav2letter++ / asrkit criterion path).

Batched ASG and CTC loss+gradient and Viterbi alignment as hand-written
sm_100a CUDA kernels behind a C-ABI (include/w2l_criterion.h), exposed with
the reference's criterion API (pkg/src/asrkit/criterion.py).
"""

from .criterion import (AsgCriterion, BatchLossOutput, CtcCriterion, LossOutput, asg_loss,
                        asg_loss_grad, asg_loss_grad_batched, collapse_path, ctc_loss,
                        ctc_loss_grad, ctc_loss_grad_batched, make_criterion, validate_target,
                        viterbi, viterbi_batched)
from .errors import (AsrkitError, ContractError, InfeasibleTargetError, NumericError,
                     TargetError, TokenError)

__version__ = "0.1.0"
