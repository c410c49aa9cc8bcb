import sys, numpy as np
sys.path[:0]=['.','tests']
import paper_2601_04185_b200 as vl
from paper_2601_04185_b200.posest import score_hypotheses
g=np.load('tests/golden/score.npz')
intr=vl.CameraIntrinsics(700.0,700.0,350.0,350.0,700,700)
got=score_hypotheses(g['R'],g['t'],g['X'],g['px'],g['w'],intr,float(g['tau']))
rel=np.abs(got-g['costs'])/np.abs(g['costs'])
print('max rel %.3e median %.3e exact %d/%d'%(rel.max(), np.median(rel), int((got==g['costs']).sum()), got.size))
